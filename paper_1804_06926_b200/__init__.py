"""B200 (sm_100a) exact triangle counting -- Python binding of libtc_b200.so.

Argument marshalling only: every step of the path (clean, orient, sort, bin,
intersect, reduce) runs in the CUDA kernels behind the C ABI declared in
``include/tc.h``.  There is no CPU fallback: if the extension is missing or no
CUDA device is present, the calls raise.

PyTorch supplies device memory and the current stream; numpy arrays / CPU
tensors are passed as host pointers (TC_HOST_PTRS) and copied by the library.
Paper: Wang, Wang, Yang, Owens, "A Comparative Study on Exact Triangle Counting
Algorithms on the GPU" (arxiv 1804.06926), Alg. 2.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["count", "count_ex", "count_shard", "orient", "clustering", "edge_support",
           "enumerate_triangles", "stats_dict", "library_path",
           "TC_CLEAN", "TC_SORTED", "TC_PER_VERTEX", "TC_HOST_PTRS", "TC_VALIDATE", "TC_PRUNE",
           "TC_ID_ORDER", "masked_spgemm", "trim_workspace", "clean_shard", "count_edges_shard",
           "VARIANT_AUTO", "VARIANT_SHORT", "VARIANT_MERGE", "VARIANT_SEARCH", "VARIANT_HASH",
           "TCError"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtc_b200.so")

TC_CLEAN, TC_SORTED, TC_PER_VERTEX, TC_HOST_PTRS, TC_VALIDATE, TC_PRUNE = 1, 2, 4, 8, 16, 32
TC_ID_ORDER = 64
VARIANT_AUTO, VARIANT_SHORT, VARIANT_MERGE, VARIANT_SEARCH, VARIANT_HASH = -1, 0, 1, 2, 3
_STATUS = {0: "TC_OK", 1: "TC_EINVAL", 2: "TC_EGRAPH", 3: "TC_ENOMEM", 4: "TC_ECUDA"}
TC_ERROR = (1 << 64) - 1


class TCError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


# tc_alloc_fn / tc_free_fn (include/tc.h): workspace hook
ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class Options(ctypes.Structure):
    _fields_ = [("short_max", ctypes.c_uint32), ("skew_ratio", ctypes.c_uint32),
                ("hub_min_dplus", ctypes.c_uint32), ("force_variant", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("prune_rounds", ctypes.c_uint32),
                ("keep_workspace", ctypes.c_uint32), ("alloc", ALLOC_FN), ("free", FREE_FN),
                ("alloc_ctx", ctypes.c_void_p), ("tiny_max_n", ctypes.c_uint32),
                ("clean_method", ctypes.c_uint32), ("graph_cache", ctypes.c_uint32),
                ("lowdeg_max", ctypes.c_uint32), ("reserved", ctypes.c_uint32 * 5)]


def _torch_raw_alloc(ctx, size, stream):
    import torch
    try:   # torch's caching allocator, current device, block tied to `stream`
        return torch._C._cuda_cudaCachingAllocator_raw_alloc(size, stream or 0)
    except Exception:   # noqa: BLE001 -- a NULL return is the hook's error signal (TC_ENOMEM)
        return None


def _torch_raw_free(ctx, ptr, stream):
    import torch
    torch._C._cuda_cudaCachingAllocator_raw_delete(ptr)


# kept alive for the life of the module (ctypes callbacks must not be collected)
_TORCH_HOOK = (ALLOC_FN(_torch_raw_alloc), FREE_FN(_torch_raw_free))
_user_hooks = []


def _hook_pair(allocator):
    """allocator: "torch" (torch's caching allocator), "library" (the library's own pool), or a
    pair of Python callables alloc(size, stream) -> int pointer and free(ptr, stream)."""
    if allocator == "torch":
        return _TORCH_HOOK
    if allocator in (None, "library"):
        return None
    a, f = allocator

    def _a(_c, size, stream):
        try:
            return a(size, stream or 0)
        except Exception:   # noqa: BLE001 -- NULL is the hook's error signal (TC_ENOMEM)
            return None

    def _f(_c, ptr, stream):
        try:
            f(ptr, stream or 0)
        except Exception:   # noqa: BLE001 -- nothing can be reported from a free
            pass

    pair = (ALLOC_FN(_a), FREE_FN(_f))
    _user_hooks.append(pair)
    del _user_hooks[:-8]   # the last few stay referenced while their calls may run
    return pair


class Stats(ctypes.Structure):
    _fields_ = [("ms_clean", ctypes.c_double), ("ms_orient", ctypes.c_double),
                ("ms_sort", ctypes.c_double), ("ms_bin", ctypes.c_double),
                ("ms_intersect", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("m_undirected", ctypes.c_uint64), ("work_W", ctypes.c_uint64),
                ("work_probe", ctypes.c_uint64), ("bytes_alg", ctypes.c_uint64),
                ("bin_edges", ctypes.c_uint64 * 4), ("skipped_edges", ctypes.c_uint64),
                ("hub_sources", ctypes.c_uint64), ("max_dplus", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64), ("h2d_bytes", ctypes.c_uint64),
                ("d2h_bytes", ctypes.c_uint64), ("table_loads", ctypes.c_uint64),
                ("bytes_hash", ctypes.c_uint64), ("ms_prune", ctypes.c_double),
                ("pruned_edges", ctypes.c_uint64), ("prune_rounds", ctypes.c_uint64),
                ("work_stage", ctypes.c_uint64), ("core_edges", ctypes.c_uint64),
                ("core_words", ctypes.c_uint64), ("bytes_core", ctypes.c_uint64)]


class ClusteringSummary(ctypes.Structure):
    _fields_ = [("triangles", ctypes.c_uint64), ("wedges", ctypes.c_uint64),
                ("transitivity", ctypes.c_double), ("avg_clustering", ctypes.c_double)]


_lib = None


def library_path() -> str:
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} is missing: run `python __graft_entry__.py` / "
                           "paper_1804_06926_b200/_build.py first (there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    u64, u32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
    lib.tc_default_options.argtypes = [ctypes.POINTER(Options)]
    lib.tc_default_options.restype = None
    lib.tc_count.argtypes = [u64, u64, vp, vp, u32]
    lib.tc_count.restype = u64
    lib.tc_count_ex.argtypes = [u64, u64, vp, vp, u32, ctypes.POINTER(Options), vp, vp,
                                ctypes.POINTER(Stats)]
    lib.tc_count_ex.restype = ctypes.c_int
    lib.tc_count_shard.argtypes = [u64, u64, vp, vp, u32, ctypes.POINTER(Options), ctypes.c_int,
                                   ctypes.c_int, vp, vp, ctypes.POINTER(Stats)]
    lib.tc_count_shard.restype = ctypes.c_int
    lib.tc_clean_shard.argtypes = [u64, u64, vp, vp, u32, ctypes.POINTER(Options), ctypes.c_int,
                                   ctypes.c_int, vp, vp, vp]
    lib.tc_clean_shard.restype = ctypes.c_int
    lib.tc_count_edges_shard.argtypes = [u64, u64, vp, vp, u32, ctypes.POINTER(Options), ctypes.c_int,
                                         ctypes.c_int, vp, vp, ctypes.POINTER(Stats)]
    lib.tc_count_edges_shard.restype = ctypes.c_int
    lib.tc_orient.argtypes = [u64, u64, vp, vp, u32, ctypes.POINTER(Options), vp, vp, vp]
    lib.tc_orient.restype = ctypes.c_int
    lib.tc_clustering.argtypes = [u64, u64, vp, vp, u32, ctypes.POINTER(Options), vp, vp,
                                  ctypes.POINTER(ClusteringSummary), ctypes.POINTER(Stats)]
    lib.tc_clustering.restype = ctypes.c_int
    lib.tc_edge_support.argtypes = [u64, u64, vp, vp, u32, ctypes.POINTER(Options), vp, vp, vp, vp,
                                    ctypes.POINTER(Stats)]
    lib.tc_edge_support.restype = ctypes.c_int
    lib.tc_enumerate.argtypes = [u64, u64, vp, vp, u32, ctypes.POINTER(Options), vp, u64, vp,
                                 ctypes.POINTER(Stats)]
    lib.tc_enumerate.restype = ctypes.c_int
    lib.tc_masked_spgemm.argtypes = [u64, u64, vp, vp, u32, ctypes.POINTER(Options), vp, vp, vp, vp,
                                     vp, ctypes.POINTER(Stats)]
    lib.tc_masked_spgemm.restype = ctypes.c_int
    lib.tc_last_error.argtypes = []
    lib.tc_last_error.restype = ctypes.c_char_p
    lib.tc_launches_issued.argtypes = []
    lib.tc_launches_issued.restype = ctypes.c_uint64
    lib.tc_trim_workspace.argtypes = [ctypes.c_int]
    lib.tc_trim_workspace.restype = ctypes.c_int
    lib.tc_version.argtypes = []
    lib.tc_version.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(status: int):
    if status != 0:
        raise TCError(status, _load().tc_last_error().decode())


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _arrays(rowptr, col):
    """-> (n, M, rowptr_ptr, col_ptr, on_device, keepalive)."""
    if _is_torch(rowptr):
        import torch
        assert rowptr.dtype in (torch.int64, torch.uint64) and col.dtype in (torch.int32, torch.uint32)
        rowptr = rowptr.contiguous()
        col = col.contiguous()
        on_dev = rowptr.is_cuda
        if on_dev != col.is_cuda:
            raise ValueError("rowptr and col must be on the same side")
        n = rowptr.numel() - 1
        M = col.numel()
        return n, M, rowptr.data_ptr(), (col.data_ptr() if M else None), on_dev, (rowptr, col)
    rowptr = np.ascontiguousarray(rowptr, dtype=np.uint64)
    col = np.ascontiguousarray(col, dtype=np.uint32)
    n = rowptr.size - 1
    return n, col.size, rowptr.ctypes.data, (col.ctypes.data if col.size else None), False, (rowptr, col)


def _flags(clean=False, sorted_rows=False, per_vertex=False, validate=False, prune=False,
           id_order=False, on_dev=True):
    return ((TC_CLEAN if clean else 0) | (TC_SORTED if sorted_rows else 0) |
            (TC_PER_VERTEX if per_vertex else 0) | (TC_VALIDATE if validate else 0) |
            (TC_PRUNE if prune else 0) | (TC_ID_ORDER if id_order else 0) |
            (0 if on_dev else TC_HOST_PTRS))


def _options(stream=None, force_variant=None, short_max=None, skew_ratio=None, hub_min_dplus=None,
             prune_rounds=None, on_device=True, allocator=None, device=None, keep_workspace=None,
             tiny_max_n=None, clean_method=None, graph_cache=None, lowdeg_max=None):
    """tc_options for one call.  Device calls default to the current stream of the inputs'
    device and to torch's caching allocator for the workspace."""
    o = Options()
    _load().tc_default_options(ctypes.byref(o))
    if stream is None and on_device:
        import torch
        stream = torch.cuda.current_stream(device).cuda_stream
    o.stream = stream or None
    if allocator is None and on_device:
        # TC_ALLOCATOR=library: the library's own pool (compute-sanitizer sees each block;
        # torch's caching allocator sub-allocates large segments); graph replay owns its
        # workspace (graph memory), so it takes no hook
        allocator = "library" if graph_cache else os.environ.get("TC_ALLOCATOR", "torch")
    hooks = _hook_pair(allocator)
    if hooks is not None:
        o.alloc, o.free = hooks
    if force_variant is not None:
        o.force_variant = force_variant
    if short_max is not None:
        o.short_max = short_max
    if skew_ratio is not None:
        o.skew_ratio = skew_ratio
    if hub_min_dplus is not None:
        o.hub_min_dplus = hub_min_dplus
    if prune_rounds is not None:
        o.prune_rounds = prune_rounds
    if keep_workspace is not None:
        o.keep_workspace = int(bool(keep_workspace))
    if tiny_max_n is not None:
        o.tiny_max_n = tiny_max_n
    if clean_method is not None:
        o.clean_method = clean_method
    if graph_cache is not None:
        o.graph_cache = int(bool(graph_cache))
    if lowdeg_max is not None:
        o.lowdeg_max = lowdeg_max
    return o


def _dev(keep, on_dev):
    return keep[0].device if on_dev else None


def _in_dev(keep, on_dev, call):
    """Run the C call with the inputs' CUDA device current (the library works on the current
    device; tc.h DEVICE)."""
    if not on_dev:
        return call()
    import torch
    with torch.cuda.device(keep[0].device):
        return call()


def stats_dict(s: Stats) -> dict:
    d = {f: getattr(s, f) for f, _ in Stats._fields_}
    d["bin_edges"] = list(s.bin_edges)
    return d


def count_ex(rowptr, col, *, clean=False, sorted_rows=False, per_vertex=False, validate=False,
             prune=False, id_order=False, stream=None, with_stats=False, **opts):
    """Triangle count of the graph (rowptr, col) [+ per-vertex counts, stats].

    torch CUDA tensors -> device pointers on the current stream; numpy arrays or
    CPU tensors -> TC_HOST_PTRS (the library copies in and out).
    """
    lib = _load()
    n, M, rp, cp, on_dev, keep = _arrays(rowptr, col)
    flags = (TC_CLEAN if clean else 0) | (TC_SORTED if sorted_rows else 0) | \
            (TC_PER_VERTEX if per_vertex else 0) | (TC_VALIDATE if validate else 0) | \
            (TC_PRUNE if prune else 0) | (TC_ID_ORDER if id_order else 0) | \
            (0 if on_dev else TC_HOST_PTRS)
    o = _options(stream=stream, on_device=on_dev, device=_dev(keep, on_dev), **opts)
    total = ctypes.c_uint64(0)
    pv = None
    pv_ptr = None
    if per_vertex:
        if on_dev:
            import torch
            pv = torch.empty(max(n, 1), dtype=torch.int64, device=keep[0].device)
            pv_ptr = pv.data_ptr()
        else:
            pv = np.zeros(max(n, 1), dtype=np.uint64)
            pv_ptr = pv.ctypes.data
    st = Stats()
    _check(_in_dev(keep, on_dev, lambda: lib.tc_count_ex(n, M, rp, cp, flags, ctypes.byref(o), ctypes.addressof(total), pv_ptr,
                           ctypes.byref(st) if with_stats else None)))
    out = [int(total.value)]
    if per_vertex:
        out.append(pv[:n])
    if with_stats:
        out.append(stats_dict(st))
    return out[0] if len(out) == 1 else tuple(out)


def count(rowptr, col, **kw):
    """Convenience: total triangle count (see count_ex for keywords)."""
    return count_ex(rowptr, col, **kw)


def count_shard(rowptr, col, rank: int, world: int, partial, *, clean=False, sorted_rows=False,
                per_vertex_partial=None, prune=False, stream=None, with_stats=False, **opts):
    """Enqueue this rank's share; `partial` is a 1-element int64 CUDA tensor (overwritten)."""
    lib = _load()
    n, M, rp, cp, on_dev, keep = _arrays(rowptr, col)
    if not on_dev:
        raise ValueError("count_shard takes CUDA tensors")
    flags = (TC_CLEAN if clean else 0) | (TC_SORTED if sorted_rows else 0) | \
            (TC_PER_VERTEX if per_vertex_partial is not None else 0) | (TC_PRUNE if prune else 0)
    o = _options(stream=stream, device=_dev(keep, on_dev), **opts)
    st = Stats()
    _check(_in_dev(keep, on_dev, lambda: lib.tc_count_shard(n, M, rp, cp, flags, ctypes.byref(o), rank, world, partial.data_ptr(),
                              per_vertex_partial.data_ptr() if per_vertex_partial is not None else None,
                              ctypes.byref(st) if with_stats else None)))
    return stats_dict(st) if with_stats else None


def clean_shard(rowptr, col, rank: int, world: int, *, stream=None, **opts):
    """Sharded a1 (tc_clean_shard): this rank's unique undirected edges as sorted int64 keys
    (min << b) | max (a CUDA tensor view of length m_r) and the degrees they contribute
    (int32[n]); sum the degrees and concatenate the edges over ranks, then count_edges_shard."""
    import torch
    lib = _load()
    n, M, rp, cp, on_dev, keep = _arrays(rowptr, col)
    if not on_dev:
        raise ValueError("clean_shard takes CUDA tensors")
    dev = keep[0].device
    edges = torch.empty(max(M, 1), dtype=torch.int64, device=dev)
    deg = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    o = _options(stream=stream, device=dev, **opts)
    m = ctypes.c_uint64(0)
    _check(_in_dev(keep, on_dev, lambda: lib.tc_clean_shard(
        n, M, rp, cp, 0, ctypes.byref(o), rank, world, edges.data_ptr(), deg.data_ptr(),
        ctypes.addressof(m))))
    return edges[:m.value], deg[:n]


def count_edges_shard(n: int, edges, degrees, rank: int, world: int, partial, *,
                      per_vertex_partial=None, id_order=False, stream=None, with_stats=False, **opts):
    """tc_count_edges_shard: this rank's share of the count from the cleaned edge list of every
    rank (int64 CUDA tensor, any order) and the summed degrees; `partial` (int64[1]) is
    overwritten."""
    lib = _load()
    edges = edges.contiguous()
    degrees = degrees.contiguous()
    keep = (edges, degrees)
    flags = (TC_PER_VERTEX if per_vertex_partial is not None else 0) | (TC_ID_ORDER if id_order else 0)
    o = _options(stream=stream, device=edges.device, **opts)
    st = Stats()
    _check(_in_dev(keep, True, lambda: lib.tc_count_edges_shard(
        n, edges.numel(), edges.data_ptr() if edges.numel() else degrees.data_ptr(),
        degrees.data_ptr(), flags, ctypes.byref(o), rank, world, partial.data_ptr(),
        per_vertex_partial.data_ptr() if per_vertex_partial is not None else None,
        ctypes.byref(st) if with_stats else None)))
    return stats_dict(st) if with_stats else None


def orient(rowptr, col, *, clean=False, sorted_rows=False, prune=False, id_order=False, stream=None,
           **opts):
    """Steps a1-a4 only: the oriented compacted CSR (off+, col+) on the input's side
    (with prune=True: of the leaf-pruned graph, NEXT-2)."""
    lib = _load()
    n, M, rp, cp, on_dev, keep = _arrays(rowptr, col)
    flags = _flags(clean, sorted_rows, False, False, prune, id_order, on_dev)
    o = _options(stream=stream, on_device=on_dev, device=_dev(keep, on_dev), **opts)
    mp = ctypes.c_uint64(0)
    if on_dev:
        import torch
        off = torch.empty(n + 1, dtype=torch.int64, device=keep[0].device)
        colp = torch.empty(max(M, 1), dtype=torch.int32, device=keep[0].device)
        _check(_in_dev(keep, on_dev, lambda: lib.tc_orient(n, M, rp, cp, flags, ctypes.byref(o), off.data_ptr(), colp.data_ptr(),
                             ctypes.addressof(mp))))
    else:
        off = np.zeros(n + 1, dtype=np.uint64)
        colp = np.zeros(max(M, 1), dtype=np.uint32)
        _check(_in_dev(keep, on_dev, lambda: lib.tc_orient(n, M, rp, cp, flags, ctypes.byref(o), off.ctypes.data, colp.ctypes.data,
                             ctypes.addressof(mp))))
    return off, colp[:mp.value]


def clustering(rowptr, col, *, clean=False, sorted_rows=False, validate=False, per_vertex=False,
               local=True, prune=False, stream=None, with_stats=False, **opts):
    """NEXT-1: (local clustering coefficients or None, summary dict[, t(v)][, stats]).

    local_cc[v] = 2t(v)/(d(v)(d(v)-1)) (0 if d(v) < 2); summary = triangles, wedges,
    transitivity = 3T/wedges, avg_clustering over all n vertices (include/tc.h).
    Outputs live on the input's side (CUDA tensors or numpy arrays).
    """
    lib = _load()
    n, M, rp, cp, on_dev, keep = _arrays(rowptr, col)
    flags = (TC_CLEAN if clean else 0) | (TC_SORTED if sorted_rows else 0) | \
            (TC_VALIDATE if validate else 0) | (TC_PRUNE if prune else 0) | \
            (0 if on_dev else TC_HOST_PTRS)
    o = _options(stream=stream, on_device=on_dev, device=_dev(keep, on_dev), **opts)
    cc = pv = None
    if on_dev:
        import torch
        dev = keep[0].device
        if local:
            cc = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        if per_vertex:
            pv = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        ptr = lambda a: a.data_ptr() if a is not None else None  # noqa: E731
    else:
        if local:
            cc = np.zeros(max(n, 1), dtype=np.float64)
        if per_vertex:
            pv = np.zeros(max(n, 1), dtype=np.uint64)
        ptr = lambda a: a.ctypes.data if a is not None else None  # noqa: E731
    summ = ClusteringSummary()
    st = Stats()
    _check(_in_dev(keep, on_dev, lambda: lib.tc_clustering(n, M, rp, cp, flags, ctypes.byref(o), ptr(cc), ptr(pv), ctypes.byref(summ),
                             ctypes.byref(st) if with_stats else None)))
    out = [cc[:n] if cc is not None else None,
           {f: getattr(summ, f) for f, _ in ClusteringSummary._fields_}]
    if per_vertex:
        out.append(pv[:n])
    if with_stats:
        out.append(stats_dict(st))
    return tuple(out)


def edge_support(rowptr, col, *, clean=False, sorted_rows=False, validate=False, prune=False,
                 stream=None, with_stats=False, **opts):
    """NEXT-3: (off+, col+, support) -- the oriented CSR exactly as orient() returns it (input
    ids, each undirected edge once, rows ascending) and the number of triangles through each
    of its edges (uint32), on the input's side [+ stats]."""
    lib = _load()
    n, M, rp, cp, on_dev, keep = _arrays(rowptr, col)
    flags = (TC_CLEAN if clean else 0) | (TC_SORTED if sorted_rows else 0) | \
            (TC_VALIDATE if validate else 0) | (TC_PRUNE if prune else 0) | \
            (0 if on_dev else TC_HOST_PTRS)
    o = _options(stream=stream, on_device=on_dev, device=_dev(keep, on_dev), **opts)
    mp = ctypes.c_uint64(0)
    st = Stats()
    if on_dev:
        import torch
        dev = keep[0].device
        off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        colp = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
        sup = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
        ptrs = (off.data_ptr(), colp.data_ptr(), sup.data_ptr())
    else:
        off = np.zeros(n + 1, dtype=np.uint64)
        colp = np.zeros(max(M, 1), dtype=np.uint32)
        sup = np.zeros(max(M, 1), dtype=np.uint32)
        ptrs = (off.ctypes.data, colp.ctypes.data, sup.ctypes.data)
    _check(_in_dev(keep, on_dev, lambda: lib.tc_edge_support(n, M, rp, cp, flags, ctypes.byref(o), *ptrs, ctypes.addressof(mp),
                               ctypes.byref(st) if with_stats else None)))
    out = (off, colp[:mp.value], sup[:mp.value])
    return out + (stats_dict(st),) if with_stats else out


def enumerate_triangles(rowptr, col, *, capacity=None, out=None, clean=False, sorted_rows=False,
                        validate=False, prune=False, stream=None, with_stats=False, **opts):
    """NEXT-3: (T, triangles) -- triangles is a (min(T, capacity), 3) array of ascending input
    ids (int32 CUDA tensor / uint32 numpy array on the input's side), unspecified row order.
    capacity=None sizes the output exactly (one counting call first); `out` = a preallocated
    contiguous (capacity, 3) 32-bit array on the input's side (capacity = len(out))."""
    lib = _load()
    n, M, rp, cp, on_dev, keep = _arrays(rowptr, col)
    flags = (TC_CLEAN if clean else 0) | (TC_SORTED if sorted_rows else 0) | \
            (TC_VALIDATE if validate else 0) | (TC_PRUNE if prune else 0) | \
            (0 if on_dev else TC_HOST_PTRS)
    o = _options(stream=stream, on_device=on_dev, device=_dev(keep, on_dev), **opts)
    total = ctypes.c_uint64(0)
    st = Stats()
    if out is not None:
        capacity = len(out)
    if capacity is None:
        _check(_in_dev(keep, on_dev, lambda: lib.tc_enumerate(n, M, rp, cp, flags, ctypes.byref(o), None, 0,
                                ctypes.addressof(total), None)))
        capacity = total.value
    if out is not None:
        tri = out
        tp = out.data_ptr() if on_dev else out.ctypes.data
    elif on_dev:
        import torch
        tri = torch.empty((max(capacity, 1), 3), dtype=torch.int32, device=keep[0].device)
        tp = tri.data_ptr()
    else:
        tri = np.zeros((max(capacity, 1), 3), dtype=np.uint32)
        tp = tri.ctypes.data
    _check(_in_dev(keep, on_dev, lambda: lib.tc_enumerate(n, M, rp, cp, flags, ctypes.byref(o), tp, capacity,
                            ctypes.addressof(total), ctypes.byref(st) if with_stats else None)))
    out = (int(total.value), tri[:min(total.value, capacity)])
    return out + (stats_dict(st),) if with_stats else out


def masked_spgemm(rowptr, col, *, id_order=False, clean=False, sorted_rows=False, validate=False,
                  prune=False, stream=None, with_stats=False, **opts):
    """NEXT-4 (Alg. 3 masked): (off_u, col_u, C, T) -- the upper triangle of A in the vertex
    order (degree, id) or plain ids (id_order=True, Fig. mm), in input ids with rows ascending,
    C = A o (L U) at each of its entries, and T = sum(C over both triangles) / 2 [+ stats]."""
    lib = _load()
    n, M, rp, cp, on_dev, keep = _arrays(rowptr, col)
    flags = _flags(clean, sorted_rows, False, validate, prune, id_order, on_dev)
    o = _options(stream=stream, on_device=on_dev, device=_dev(keep, on_dev), **opts)
    nnz = ctypes.c_uint64(0)
    total = ctypes.c_uint64(0)
    st = Stats()
    if on_dev:
        import torch
        dev = keep[0].device
        off = torch.empty(n + 1, dtype=torch.int64, device=dev)
        colp = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
        c = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
        ptrs = (off.data_ptr(), colp.data_ptr(), c.data_ptr())
    else:
        off = np.zeros(n + 1, dtype=np.uint64)
        colp = np.zeros(max(M, 1), dtype=np.uint32)
        c = np.zeros(max(M, 1), dtype=np.uint32)
        ptrs = (off.ctypes.data, colp.ctypes.data, c.ctypes.data)
    _check(_in_dev(keep, on_dev, lambda: lib.tc_masked_spgemm(n, M, rp, cp, flags, ctypes.byref(o), *ptrs, ctypes.addressof(nnz),
                                ctypes.addressof(total), ctypes.byref(st) if with_stats else None)))
    out = (off, colp[:nnz.value], c[:nnz.value], int(total.value))
    return out + (stats_dict(st),) if with_stats else out


def trim_workspace(device: int = -1) -> None:
    """Return the library pool's cached workspace on `device` to the driver (tc_trim_workspace)."""
    _check(_load().tc_trim_workspace(device))


def version() -> str:
    return _load().tc_version().decode()


def launches_issued() -> int:
    """tc_launches_issued: kernels launched so far by this thread's library calls."""
    return int(_load().tc_launches_issued())
