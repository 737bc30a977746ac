"""bench.py -- exact triangle counting on B200: ms and edges/s on R-MAT, % of HBM roofline.

Contract (driver): `python bench.py --gpus N --steps K --warmup W [--impl reference]`; for
N > 1 launched under torch.distributed.run (one rank per GPU, NCCL).  Rank 0 prints ONE
JSON line.

A step = one pass of the whole hot path (plus a8 for N > 1)
over the workload's RAW arcs (duplicates, self-loops, one-directional arcs): clean ->
orient -> bin -> intersect -> reduce, i.e. one tc_count_ex call (tc_count_shard + one
NCCL allreduce of the uint64 count per rank for N > 1).  Inputs are resident in HBM when
the timed region starts; L2 is flushed (a 512 MiB write) between timed steps, outside the
per-step CUDA-event spans.  `value` = undirected edges m / (ms per step), whole job.

Workload at N = 1: BASELINE.json configs[1], R-MAT scale 21 edge factor 16 (Graph500
A,B,C,D = .57,.19,.19,.05), seeded and synthetic.  For N > 1 the
same graph is replicated on every rank and the sources are split by work (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "triangle-count ms and edges/s on R-MAT s21–24 @1/2/4/8 B200; % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--scale", type=int, default=21)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the NEXT-row measurements")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"   # B200_PROFILING.md fallback figure


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm / cpu baseline
def oracle_run(g):
    """The CPU oracle (oracle/, test infrastructure) on the whole graph; returns (T, m, seconds)."""
    import oracle
    t0 = time.perf_counter()
    T, st = oracle.count(g.n, g.rowptr, g.col, with_stats=True)
    return T, st["m"], time.perf_counter() - t0


def cpu_baseline(g, m):
    import oracle
    T, m_o, sec = oracle_run(g)
    return {"value": m_o / sec, "unit": "edges/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"whole workload ({g.name}, {g.arcs} raw arcs, m={m_o}), one run of the "
                      f"oracle's clean+orient+forward, {sec:.2f} s", "seconds": sec, "T": T}


def reference_arm(args, g, rank, world):
    """--impl reference: the oracle as it stands, timed on the host cores (rank 0 only)."""
    if rank != 0:
        return None
    import oracle
    K, W = args.steps, args.warmup
    # bounded sample: one step = the oracle on the whole workload (about 8-30 s of CPU work
    # at s21 on a 16-core host).  W and K are honoured as requested unless the run would
    # exceed ~5 minutes; then K alone is reduced (and the note says so).
    budget_s = 300.0
    first = oracle_run(g)[2] if W > 0 else None
    w_eff = W
    for _ in range(max(W - 1, 0)):
        oracle_run(g)
    est = first if first else 10.0
    k_eff = max(1, min(K, int((budget_s - W * est) / est)))
    secs, T, m = [], None, None
    for _ in range(k_eff):
        T, m, s = oracle_run(g)
        secs.append(s)
    sec = sum(secs) / len(secs)
    value = m / sec
    return {"metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": k_eff,
            "warmup": w_eff, "ms_per_step": 1e3 * sec, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic", "impl": "reference",
            "config": {"workload": g.name, "n": g.n, "m": m, "raw_arcs": g.arcs, "T": T,
                       "note": (f"requested steps={K} warmup={W}" + ("" if k_eff == K else
                                f"; steps reduced to {k_eff} to stay within {budget_s:.0f} s") +
                                "; each step = the oracle on the whole workload")},
            "cpu_baseline": {"value": value, "unit": "edges/s", "cores": oracle.num_threads(),
                             "kind": "oracle", "sample": f"whole workload per step ({g.name})"},
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _timed(torch, flush, stream, fn, reps=3):
    """Mean CUDA-event ms of fn() over reps calls (L2 flushed before each), last result."""
    fn()
    tot, out = 0.0, None
    for _ in range(reps):
        flush.fill_(3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = fn()
        b.record(stream)
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps, out


def clean_input_ms(tc, torch, rp, cl, flush, stream, T):
    """SURVEY §8(d)'s own definition of the headline ms: from a CLEAN symmetric CSR resident on
    the device (TC_CLEAN | TC_SORTED: a1 skipped) to the count.  The clean CSR is prepared
    outside the timed region from the library's oriented CSR (torch sort: input plumbing)."""
    n = rp.numel() - 1
    off, colp = tc.orient(rp, cl)
    src = torch.repeat_interleave(torch.arange(n, device=rp.device), off[1:] - off[:-1])
    dst = colp.to(torch.int64)
    b = max(1, (n - 1).bit_length())
    keys = torch.cat([(src << b) | dst, (dst << b) | src])
    keys, _ = torch.sort(keys)
    s2, d2 = keys >> b, keys & ((1 << b) - 1)
    crp = torch.zeros(n + 1, dtype=torch.int64, device=rp.device)
    crp[1:] = torch.cumsum(torch.bincount(s2, minlength=n), 0)
    ccl = d2.to(torch.int32).contiguous()
    del off, colp, src, dst, keys, s2, d2
    ms, (Tc, st) = _timed(torch, flush, stream,
                          lambda: tc.count_ex(crp, ccl, clean=True, sorted_rows=True, with_stats=True))
    assert Tc == T
    return {"ms_per_call": ms, "edges_per_s": st["m_undirected"] / (ms * 1e-3),
            "phases_ms": {k: st[k] for k in ("ms_orient", "ms_bin", "ms_intersect")},
            "call": "tc_count_ex(TC_CLEAN | TC_SORTED) on the symmetric sorted CSR (a2-a7; a1 skipped)"}


def next_rows_23(tc, torch, np, graphgen, rp, cl, flush, stream, m, T, count_ms):
    """NEXT-2 / NEXT-3 timed through their C-ABI calls, device pointers."""
    rows = {}
    # NEXT-3 edge support on the bench workload
    sms, (off, colp, sup) = _timed(torch, flush, stream, lambda: tc.edge_support(rp, cl))
    assert int(sup.to(torch.int64).sum().item()) == 3 * T
    rows["NEXT-3 edge support"] = {
        "ms_per_call": sms, "edges_per_s": m / (sms * 1e-3), "overhead_vs_count_ms": sms - count_ms,
        "max_support": int(sup.max().item()),
        "call": "tc_edge_support: count crediting all three edges of every triangle + the "
                "oriented CSR and supports mapped back to input ids"}
    del off, colp, sup
    # NEXT-3 enumeration: output-bound (12 B per triangle)
    tri = torch.empty((T, 3), dtype=torch.int32, device=rp.device)
    ems, (Te, _) = _timed(torch, flush, stream, lambda: tc.enumerate_triangles(rp, cl, out=tri))
    assert Te == T
    rows["NEXT-3 enumeration"] = {
        "ms_per_call": ems, "triangles_per_s": T / (ems * 1e-3), "output_bytes": 12 * T,
        "output_GB_per_s": 12 * T / (ems * 1e-3) / 1e9,
        "call": "tc_enumerate into a preallocated device buffer of T triples (capacity = T)"}
    del tri
    # NEXT-4 masked SpGEMM (Alg. 3): C = A o (L U) at the upper-triangle nonzeros
    mms, (_, _, cvals, Tm) = _timed(torch, flush, stream, lambda: tc.masked_spgemm(rp, cl))
    assert Tm == T and int(cvals.to(torch.int64).sum().item()) == T
    rows["NEXT-4 masked SpGEMM"] = {
        "ms_per_call": mms, "edges_per_s": m / (mms * 1e-3), "overhead_vs_count_ms": mms - count_ms,
        "max_C": int(cvals.max().item()),
        "call": "tc_masked_spgemm (rank order, Alg. 3 line 1): C at each upper-triangle entry "
                "mapped back to input ids"}
    del cvals
    # NEXT-2 leaf pruning where it matters: the road mesh (BASELINE configs[3])
    g = graphgen.road_mesh()
    rrp = torch.from_numpy(g.rowptr.view(np.int64)).to(rp.device)
    rcl = torch.from_numpy(g.col.view(np.int32)).to(rp.device)
    bms, (Tb, sb) = _timed(torch, flush, stream, lambda: tc.count_ex(rrp, rcl, with_stats=True))
    out = {"workload": g.name, "count_ms_unpruned": bms, "m": sb["m_undirected"]}
    for r in (1, 2, 0):
        pms, (Tp, sp) = _timed(torch, flush, stream,
                               lambda: tc.count_ex(rrp, rcl, prune=True, prune_rounds=r, with_stats=True))
        assert Tp == Tb
        out[f"rounds={r or 'fixed-point'}"] = {
            "ms_per_call": pms, "prune_ms": sp["ms_prune"], "pruned_edges": sp["pruned_edges"],
            "rounds_run": sp["prune_rounds"], "edges_per_s": sb["m_undirected"] / (pms * 1e-3)}
    rows["NEXT-2 leaf pruning (road mesh)"] = out
    return rows


# ------------------------------------------------------------------ native arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import numpy as np
    import graphgen

    g = graphgen.rmat(args.scale, args.edge_factor)
    if args.impl == "reference":
        line = reference_arm(args, g, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import torch
    import paper_1804_06926_b200 as tc
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    rp = torch.from_numpy(g.rowptr.view(np.int64)).to(dev)
    cl = torch.from_numpy(g.col.view(np.int32)).to(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    partial = torch.zeros(1, dtype=torch.int64, device=dev)

    def step(with_stats=False):
        if world == 1:
            return tc.count_ex(rp, cl, with_stats=with_stats)
        st = tc.count_shard(rp, cl, rank, world, partial, with_stats=with_stats)
        dist.all_reduce(partial)
        return (int(partial.item()), st) if with_stats else int(partial.item())

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, per-step CUDA events, L2 flushed between steps
    sampler = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    stats = []
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    T_total = None
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        ev[k][0].record(stream)
        out = step(with_stats=True)
        ev[k][1].record(stream)
        T_total, st = out
        stats.append(st)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / len(step_ms)
    ix_ms = sum(s["ms_intersect"] for s in stats) / len(stats)
    bin_ms = sum(s["ms_bin"] for s in stats) / len(stats)
    if dist is not None:
        t = torch.tensor([ms, ix_ms, bin_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ix_ms, bin_ms = t.tolist()
    st = stats[-1]
    m = st["m_undirected"]
    launches = st["kernel_launches"] * args.steps

    # ---- end to end through the public API with HOST buffers (pinned), N = 1 semantics per rank
    e2e = None
    if not args.no_e2e:
        rp_h = torch.from_numpy(g.rowptr.view(np.int64)).pin_memory()
        cl_h = torch.from_numpy(g.col.view(np.int32)).pin_memory()
        tc.count_ex(rp_h, cl_h)   # warm
        reps = max(3, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(reps):
            got = tc.count_ex(rp_h, cl_h, with_stats=True)
        e2e_s = (time.perf_counter() - t0) / reps
        assert got[0] == T_total
        e2e = {"value": m / e2e_s, "unit": "edges/s", "ms_per_step": 1e3 * e2e_s,
               "h2d_bytes_per_step": got[1]["h2d_bytes"], "d2h_bytes_per_step": got[1]["d2h_bytes"],
               "note": "tc_count_ex with TC_HOST_PTRS from pinned host memory: H2D of the raw CSR, "
                       "the whole path, D2H of the count; host wall clock, single GPU per rank"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    peak, peak_kind = load_peaks()
    b_alg = st["bytes_alg"]
    b_hash = st["bytes_hash"]
    achieved = b_hash / (ix_ms * 1e-3) / 1e9 / world  # GB/s per GPU
    achieved_alg = b_alg / (ix_ms * 1e-3) / 1e9 / world
    line = {
        "metric": METRIC, "value": m / (ms * 1e-3), "unit": "edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded R-MAT, Graph500 A,B,C,D=.57,.19,.19,.05; raw arcs)",
        "config": {"workload": g.name, "n": g.n, "m": m, "raw_arcs": g.arcs, "T": T_total,
                   "parallelism": f"replicated graph, work-split sources x{world}",
                   "l2": "flushed between timed steps (512 MiB write outside the event spans)",
                   "step": "tc_count_ex on raw arcs: clean, orient, bin, intersect, reduce"
                           + (" + NCCL allreduce" if world > 1 else "")},
        "phases_ms": {k: sum(s[k] for s in stats) / len(stats)
                      for k in ("ms_clean", "ms_orient", "ms_sort", "ms_bin", "ms_intersect", "ms_total")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "kernel": "a6+a7 intersection phase (k_hash_cta bitmap + hash, k_hash_warp "
                               "[+ empty SHORT/MERGE/SEARCH launches]), CUDA events on the launch stream",
                     "bytes_model": "B_hash = 4*sum min(|N+(u)>v|, d+v) + 8*HASH edges + 4*table loads "
                                    "(bytes the implemented a6 must read; DESIGN.md sec. 5)",
                     "bytes_hash": b_hash, "kernel_ms": ix_ms, "bin_ms": bin_ms, "peak_kind": peak_kind,
                     "survey_B_alg": {"bytes": b_alg, "model": "4W + 16m (SURVEY.md 8(d), merge-based)",
                                      "achieved": achieved_alg, "frac": achieved_alg / peak,
                                      "frac_incl_binning": b_alg / ((ix_ms + bin_ms) * 1e-3) / 1e9 / world / peak},
                     "survey_B_stage": {"bytes": 4 * (m + st["work_stage"]) + 16 * m,
                                        "model": "4(m + sum d-(v) d+(v)) + 16m (SURVEY.md 8(d))",
                                        "frac": (4 * (m + st["work_stage"]) + 16 * m)
                                                / (ix_ms * 1e-3) / 1e9 / world / peak},
                     "work_W": st["work_W"], "work_probe": st["work_probe"],
                     "table_loads": st["table_loads"]},
        "gpu_launches": launches,
        "e2e": e2e,
        "clocks": clocks,
    }
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            tr = json.load(open(tf)).get(g.name)
            if tr:
                line["roofline"]["traffic"] = tr["dram_bytes_per_launch"]
                line["roofline"]["traffic_source"] = tr["source"]
                for k in ("bitmap_kernel_l2_hit_pct", "bitmap_kernel_dram_throughput_pct"):
                    if tr.get(k) is not None:
                        line["roofline"][k] = tr[k]
        except (OSError, ValueError):
            pass
    if world == 1 and not args.no_next:
        # NEXT-1: clustering coefficients + transitivity on the same
        # workload through tc_clustering (count with t(v), then the c(v) kernel)
        cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(3)]
        tc.clustering(rp, cl)
        for a, b in cev:
            flush.fill_(1)
            a.record(stream)
            _, summ = tc.clustering(rp, cl)
            b.record(stream)
        torch.cuda.synchronize()
        cms = sum(a.elapsed_time(b) for a, b in cev) / len(cev)
        assert summ["triangles"] == T_total
        line["next_rows"] = {"NEXT-1 clustering": {
            "ms_per_call": cms, "edges_per_s": m / (cms * 1e-3), "overhead_vs_count_ms": cms - ms,
            "transitivity": summ["transitivity"], "avg_clustering": summ["avg_clustering"],
            "wedges": summ["wedges"],
            "call": "tc_clustering (device pointers): count with per-vertex t(v) + local c(v) for all n"}}
        line["survey_clean_input"] = clean_input_ms(tc, torch, rp, cl, flush, stream, T_total)
        line["next_rows"].update(next_rows_23(tc, torch, np, graphgen, rp, cl, flush, stream, m,
                                              T_total, ms))
    if world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(g, m)
        assert cb.pop("T") == T_total, "oracle and CUDA path disagree"
        line["cpu_baseline"] = cb
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
