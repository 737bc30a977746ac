"""Multi-GPU with a2-a5 sharded (csrc/shard.cu, include/tc.h "Sharded pipeline"), round 2.

The phases of one rank, each a C call (argument marshalling only), between the collectives:

    clean_shard            (a1 on the rank's edges)      -> all-reduce degrees
    shard_orient           (ranks, own edges oriented)   -> all-reduce d+
    shard_partition        (off+, row ranges, pairs)     -> all-to-all pairs
    shard_rows             (the rank's rows of col+)     -> all-gather col+ (G broadcasts)
    shard_work             (a5 on the rank's rows)       -> all-reduce owner entries / lengths
    shard_route            (owner split, HASH entries)   -> all-to-all entries
    shard_count            (owners, tasks, a6 + a7)      -> all-reduce the count

``run_rank`` drives one rank against a ``Comm`` (dist.py's NCCL one); ``emulate`` runs every
rank of a world in ONE process on one GPU, phase by phase, doing the collectives with local
tensor operations and timing every rank's phases with CUDA events -- the projection and the
parity tests of the sharded path (a GPU cannot run ranks that wait on each other).
"""
from __future__ import annotations

import ctypes
import os

from . import (TC_ID_ORDER, TC_PER_VERTEX, _check, _load, _options, clean_shard)

_SIG = False


def _lib():
    global _SIG
    lib = _load()
    if not _SIG:
        u64, u32, vp, i = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_int
        from . import Options
        po = ctypes.POINTER(Options)
        lib.tc_shard_orient.argtypes = [u64, u64, vp, vp, u32, po, vp, vp, vp, vp]
        lib.tc_shard_partition.argtypes = [u64, u64, vp, vp, vp, po, i, i, vp, vp, vp, vp, vp]
        lib.tc_shard_rows.argtypes = [u64, u64, vp, po, u64, vp]
        lib.tc_shard_work.argtypes = [u64, vp, vp, vp, u32, po, u64, u64, u64, u64, vp, vp, vp]
        lib.tc_shard_route.argtypes = [u64, vp, vp, vp, vp, vp, vp, u32, po, i, i, u64, u64, vp, vp]
        lib.tc_shard_count.argtypes = [u64, u64, vp, vp, vp, vp, u64, vp, u32, po, i, i, u64, u64,
                                       vp, vp, ctypes.POINTER(ctypes.c_double)]
        for f in ("tc_shard_orient", "tc_shard_partition", "tc_shard_rows", "tc_shard_work",
                  "tc_shard_route", "tc_shard_count"):
            getattr(lib, f).restype = ctypes.c_int
        _SIG = True
    return lib


def _ptr(t):
    return t.data_ptr() if t is not None and t.numel() else None


def _u64s(k):
    return (ctypes.c_uint64 * k)()


def shard_orient(n, edges, deg, *, id_order=False, stream=None, **opts):
    """P1: newid (int32[n]), the rank's edges oriented as (src, dst) rank ids, d+ partials."""
    import torch
    dev = deg.device
    m = edges.numel()
    newid = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    src = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    dst = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    dplus = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    o = _options(stream=stream, device=dev, **opts)
    _check(_lib().tc_shard_orient(n, m, _ptr(edges), _ptr(deg), TC_ID_ORDER if id_order else 0,
                                  ctypes.byref(o), _ptr(newid), _ptr(src), _ptr(dst), _ptr(dplus)))
    return newid[:n], src[:m], dst[:m], dplus[:n]


def shard_partition(n, src, dst, dplus, rank, world, *, stream=None, **opts):
    """P2: off+ (int64[n+1]), the pairs grouped by the row range of their source (int64: src |
    dst << 32), per-destination counts, row bounds and col+ bounds of every range."""
    import torch
    dev = dplus.device
    m = src.numel()
    off = torch.empty(n + 1, dtype=torch.int64, device=dev)
    pairs = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
    cnt, rb, cb = _u64s(world), _u64s(world + 1), _u64s(world + 1)
    o = _options(stream=stream, device=dev, **opts)
    _check(_lib().tc_shard_partition(n, m, _ptr(src), _ptr(dst), _ptr(dplus), ctypes.byref(o), rank,
                                     world, _ptr(off), _ptr(pairs), cnt, rb, cb))
    return off, pairs[:m], list(cnt), list(rb), list(cb)


def shard_rows(n, pairs, col_plus, col_begin, *, stream=None, **opts):
    """P3: the received pairs sorted into col_plus[col_begin : col_begin + len(pairs)]."""
    o = _options(stream=stream, device=col_plus.device, **opts)
    _check(_lib().tc_shard_rows(n, pairs.numel(), _ptr(pairs), ctypes.byref(o), col_begin,
                                col_plus.data_ptr()))


def shard_work(n, off, col_plus, dplus, row_begin, row_end, e_begin, e_end, *, per_vertex=False,
               stream=None, **opts):
    """P4: per-owner HASH entries (int32[n]) and probe lengths (int64[n]) of edges
    [e_begin, e_end), and the rank spans of rows [row_begin, row_end) (int32[n]) -- partials:
    all-reduce them."""
    import torch
    dev = off.device
    cnt = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    ln = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    sp = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    o = _options(stream=stream, device=dev, **opts)
    _check(_lib().tc_shard_work(n, off.data_ptr(), col_plus.data_ptr(), dplus.data_ptr(),
                                TC_PER_VERTEX if per_vertex else 0, ctypes.byref(o), row_begin, row_end,
                                e_begin, e_end, cnt.data_ptr(), ln.data_ptr(), sp.data_ptr()))
    return cnt[:n], ln[:n], sp[:n]


def shard_route(n, off, col_plus, dplus, cnt, ln, spans, rank, world, e_begin, e_end, *, per_vertex=False,
                stream=None, **opts):
    """P5: the HASH probe entries of edges [e_begin, e_end) grouped by their owner's rank
    (int32 triples: owner, other endpoint, CSR index | out-part flag << 31) and their counts."""
    import torch
    dev = off.device
    ent = torch.empty(3 * max(e_end - e_begin, 1), dtype=torch.int32, device=dev)
    sc = _u64s(world)
    o = _options(stream=stream, device=dev, **opts)
    _check(_lib().tc_shard_route(n, off.data_ptr(), col_plus.data_ptr(), dplus.data_ptr(), cnt.data_ptr(),
                                 ln.data_ptr(), spans.data_ptr(), TC_PER_VERTEX if per_vertex else 0, ctypes.byref(o), rank,
                                 world, e_begin, e_end, ent.data_ptr(), sc))
    counts = list(sc)
    return ent[:3 * sum(counts)], counts


def shard_count(n, off, col_plus, dplus, newid, entries, rank, world, e_begin, e_end, partial, *,
                per_vertex_partial=None, stream=None, a6_ms=None, **opts):
    """P6: this rank's share of the count into partial (int64[1], overwritten) [and t(v)
    partials in input ids into per_vertex_partial (int64[n], overwritten)].  a6_ms: a list that
    receives the a6 kernels' CUDA-event span."""
    m = col_plus.numel()
    ms = ctypes.c_double(0.0)
    o = _options(stream=stream, device=off.device, **opts)
    flags = TC_PER_VERTEX if per_vertex_partial is not None else 0
    _check(_lib().tc_shard_count(n, m, off.data_ptr(), col_plus.data_ptr(), dplus.data_ptr(),
                                 _ptr(newid), entries.numel() // 3, _ptr(entries), flags, ctypes.byref(o),
                                 rank, world, e_begin, e_end, partial.data_ptr(),
                                 _ptr(per_vertex_partial), ctypes.byref(ms) if a6_ms is not None else None))
    if a6_ms is not None:
        a6_ms.append(ms.value)


# ---------------------------------------------------------------- one rank against a Comm
def run_rank(rowptr, col, rank, world, comm, *, per_vertex=False, times=None, **opts):
    """The whole sharded count on one rank; `comm` provides all_reduce(t), all_to_all(send,
    counts, width) -> recv, broadcast_slices(col_plus, bounds).  Returns the partial count
    (int64[1]) [and the per-vertex partials] BEFORE the final all-reduce.  With a `times` dict,
    each phase's CUDA-event ms (on the current stream; the phases are synchronous) is added
    under its name, the collectives' under "comm"."""
    import torch
    n = rowptr.numel() - 1
    dev = rowptr.device
    marks = []

    def mark(name):
        if times is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((name, e))

    mark("start")
    edges, deg = clean_shard(rowptr, col, rank, world, **opts)
    mark("clean")
    comm.all_reduce(deg)
    mark("comm")
    newid, src, dst, dplus = shard_orient(n, edges, deg, **opts)
    mark("orient")
    comm.all_reduce(dplus)
    mark("comm")
    off, pairs, cnt, rb, cb = shard_partition(n, src, dst, dplus, rank, world, **opts)
    mark("partition")
    recv = comm.all_to_all(pairs, cnt, 1)
    mark("comm")
    col_plus = torch.empty(max(cb[world], 1), dtype=torch.int32, device=dev)
    shard_rows(n, recv, col_plus, cb[rank], **opts)
    mark("rows")
    # the col+ all-gather runs while this rank bins its own rows (work / route read only them)
    pending = comm.broadcast_slices(col_plus, cb, async_op=True)
    mark("comm")
    e0, e1 = cb[rank], cb[rank + 1]
    ecnt, elen, spans = shard_work(n, off, col_plus, dplus, rb[rank], rb[rank + 1], e0, e1,
                                   per_vertex=per_vertex, **opts)
    mark("work")
    comm.all_reduce(ecnt)
    comm.all_reduce(elen)
    comm.all_reduce(spans)
    mark("comm")
    ent, sc = shard_route(n, off, col_plus, dplus, ecnt, elen, spans, rank, world, e0, e1,
                          per_vertex=per_vertex, **opts)
    mark("route")
    rent = comm.all_to_all(ent, sc, 3)
    comm.wait(pending)
    mark("comm")
    partial = torch.zeros(1, dtype=torch.int64, device=dev)
    pv = torch.zeros(n, dtype=torch.int64, device=dev) if per_vertex else None
    shard_count(n, off, col_plus[:cb[world]], dplus, newid, rent, rank, world, e0, e1, partial,
                per_vertex_partial=pv, **opts)
    mark("count")
    if times is not None:
        torch.cuda.synchronize()
        for (_, a), (name, b) in zip(marks, marks[1:]):
            times[name] = times.get(name, 0.0) + a.elapsed_time(b)
    return partial, pv


# ---------------------------------------------------------------- one-GPU emulation
# Collective costs charged in the projection: B200_PROFILING.md's measured NVLink figures
# (all-gather / broadcast 770 GB/s per direction per GPU, all-reduce bus 725 GB/s); an
# all-to-all moves (world - 1) / world of each rank's send buffer over its link.
NVLINK_GATHER = 770e9
NVLINK_REDUCE = 725e9


def emulate(rowptr, col, world, *, per_vertex=False, timed=False, **opts):
    """Every rank of `world` in this process on one GPU, phase by phase; the collectives are
    local tensor operations.  Returns (total, per-vertex counts or None, report) where report
    holds each phase's per-rank CUDA-event ms and the modelled collective ms when `timed`."""
    import torch
    n = rowptr.numel() - 1
    dev = rowptr.device
    G = world
    rep = {"phases": {}, "collectives": {}}

    def run(name, fn, r):
        if not timed:
            return fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        rep["phases"].setdefault(name, [0.0] * G)[r] += a.elapsed_time(b)
        return out

    def coll(name, ms):
        rep["collectives"][name] = rep["collectives"].get(name, 0.0) + ms

    cl = [run("clean", lambda r=r: clean_shard(rowptr, col, r, G, **opts), r) for r in range(G)]
    deg = sum(d.to(torch.int64) for _, d in cl).to(torch.int32)
    coll("all-reduce degrees", 4.0 * n * 2 * (G - 1) / G / NVLINK_REDUCE * 1e3)
    p1 = [run("orient", lambda r=r: shard_orient(n, cl[r][0], deg, **opts), r) for r in range(G)]
    dplus = sum(p[3].to(torch.int64) for p in p1).to(torch.int32)
    coll("all-reduce d+", 4.0 * n * 2 * (G - 1) / G / NVLINK_REDUCE * 1e3)
    newid = p1[0][0]
    p2 = [run("partition", lambda r=r: shard_partition(n, p1[r][1], p1[r][2], dplus, r, G, **opts), r)
          for r in range(G)]
    off, rows, cb = p2[0][0], p2[0][3], p2[0][4]
    recv = []
    for q in range(G):   # destination q gets every rank's chunk q
        parts = []
        for r in range(G):
            c = p2[r][2]
            s0 = sum(c[:q])
            parts.append(p2[r][1][s0:s0 + c[q]])
        recv.append(torch.cat(parts) if parts else torch.empty(0, dtype=torch.int64, device=dev))
    coll("all-to-all pairs", max(8.0 * p[1].numel() * (G - 1) / G for p in p2) / NVLINK_GATHER * 1e3)
    del p1, p2
    col_plus = torch.empty(max(cb[G], 1), dtype=torch.int32, device=dev)
    for r in range(G):   # one shared buffer: the all-gather is implicit
        run("rows", lambda r=r: shard_rows(n, recv[r], col_plus, cb[r], **opts), r)
    coll("all-gather col+", 4.0 * cb[G] * (G - 1) / G / NVLINK_GATHER * 1e3)
    del recv
    w = [run("work", lambda r=r: shard_work(n, off, col_plus, dplus, rows[r], rows[r + 1], cb[r], cb[r + 1],
                                             per_vertex=per_vertex, **opts), r) for r in range(G)]
    ecnt = sum(x[0].to(torch.int64) for x in w).to(torch.int32)
    elen = sum(x[1] for x in w)
    spans = sum(x[2].to(torch.int64) for x in w).to(torch.int32)
    del w
    coll("all-reduce owner work", 16.0 * n * 2 * (G - 1) / G / NVLINK_REDUCE * 1e3)
    rt = [run("route", lambda r=r: shard_route(n, off, col_plus, dplus, ecnt, elen, spans, r, G, cb[r],
                                                cb[r + 1], per_vertex=per_vertex, **opts), r) for r in range(G)]
    rent = []
    for q in range(G):
        parts = []
        for r in range(G):
            c = rt[r][1]
            s0 = 3 * sum(c[:q])
            parts.append(rt[r][0][s0:s0 + 3 * c[q]])
        rent.append(torch.cat(parts))
    coll("all-to-all entries", max(4.0 * x[0].numel() * (G - 1) / G for x in rt) / NVLINK_GATHER * 1e3)
    del rt
    total, pv_sum = 0, torch.zeros(n, dtype=torch.int64, device=dev) if per_vertex else None
    prof = int(os.environ.get("TC_PROFILE_COUNT_RANK", "-1"))   # ncu --profile-from-start off
    for r in range(G):
        partial = torch.zeros(1, dtype=torch.int64, device=dev)
        pv = torch.zeros(n, dtype=torch.int64, device=dev) if per_vertex else None
        if r == prof:
            torch.cuda.profiler.start()
        a6 = [] if timed else None
        run("count", lambda r=r: shard_count(n, off, col_plus[:cb[G]], dplus, newid, rent[r], r, G, cb[r],
                                             cb[r + 1], partial, per_vertex_partial=pv, a6_ms=a6, **opts), r)
        if timed:
            rep.setdefault("a6_ms", [0.0] * G)[r] = a6[0]
        if r == prof:
            torch.cuda.profiler.stop()
        total += int(partial.item())
        if per_vertex:
            pv_sum += pv
    coll("all-reduce count", 8.0 * (n + 1 if per_vertex else 1) * 2 * (G - 1) / G / NVLINK_REDUCE * 1e3)
    if timed:
        rep["step_ms"] = sum(max(v) for v in rep["phases"].values()) + sum(rep["collectives"].values())
        # the col+ all-gather overlaps work + route + their collectives (run_rank issues it async)
        hidden = min(rep["collectives"]["all-gather col+"],
                     max(rep["phases"]["work"]) + max(rep["phases"]["route"]) +
                     rep["collectives"]["all-reduce owner work"] + rep["collectives"]["all-to-all entries"])
        rep["step_ms_overlapped"] = rep["step_ms"] - hidden
        rep["slowest_rank_ms"] = max(sum(v[r] for v in rep["phases"].values()) for r in range(G))
    return total, pv_sum, rep
