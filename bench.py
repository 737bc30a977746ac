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
Without torchrun's environment, `--gpus N` (N > 1) re-launches itself under
torch.distributed.run (one rank per GPU, 127.0.0.1 rendezvous).
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
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the road mesh / Chung-Lu / clique-union rows (other_configs)")
    ap.add_argument("--replicated-a1", action="store_true",
                    help="N > 1: every rank runs a1-a5 on the whole graph, tc_count_shard (round 1)")
    ap.add_argument("--sharded-a1-only", action="store_true",
                    help="N > 1: only the cleaning step split over the ranks (tc_clean_shard, "
                         "all-gather of the edges, tc_count_edges_shard); default: a1-a5 all "
                         "sharded (shard.py / csrc/shard.cu)")
    ap.add_argument("--one-call", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--clean-input", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--no-projection", action="store_true",
                    help="skip the one-GPU multi-GPU projection (shard.emulate) of the N = 1 line")
    ap.add_argument("--no-ncu", action="store_true",
                    help="skip the ncu DRAM-traffic capture of the a6 kernels (roofline.traffic)")
    return ap.parse_args()


def self_spawn(args) -> int:
    """`python bench.py --gpus N` without torchrun's environment: re-launch under
    torch.distributed.run with N ranks on this node (the driver's own launch line)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


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


def host_cpu():
    """lscpu model / sockets / cores / threads of the host the oracle runs on."""
    info = {}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)"):
                info[k] = v
    except (OSError, subprocess.SubprocessError):
        pass
    info["OMP_NUM_THREADS"] = os.environ.get("OMP_NUM_THREADS")
    return info


SINGLE_THREAD_SAMPLE = (18, 16)   # R-MAT s18 ef16: ~10 s of one core


def oracle_single_thread():
    """The paper's sequential-forward analogue (SURVEY §8(d) oracle timing (ii)): the oracle
    with ONE thread, in a child process (OpenMP reads OMP_NUM_THREADS at start-up), on a
    bounded sample of the same generator."""
    code = ("import sys, time; sys.path.insert(0, %r); import graphgen, oracle\n"
            "g = graphgen.rmat(%d, %d); t0 = time.perf_counter()\n"
            "T, st = oracle.count(g.n, g.rowptr, g.col, with_stats=True)\n"
            "print(time.perf_counter() - t0, st['m'], T, oracle.num_threads())"
            % (ROOT, *SINGLE_THREAD_SAMPLE))
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                             timeout=240, env=env).stdout.split()
        sec, m, T, thr = float(out[0]), int(out[1]), int(out[2]), int(out[3])
    except (OSError, subprocess.SubprocessError, ValueError, IndexError):
        return None
    return {"value": m / sec, "unit": "edges/s", "cores": thr, "seconds": sec, "T": T,
            "sample": "rmat-s%d-ef%d (whole graph), one run, OMP_NUM_THREADS=1" % SINGLE_THREAD_SAMPLE}


def cpu_baseline(g, m):
    import oracle
    T, m_o, sec = oracle_run(g)
    return {"value": m_o / sec, "unit": "edges/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"whole workload ({g.name}, {g.arcs} raw arcs, m={m_o}), one run of the "
                      f"oracle's clean+orient+forward, {sec:.2f} s", "seconds": sec, "T": T,
            "host": host_cpu(), "single_thread": oracle_single_thread()}


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
                             "kind": "oracle", "sample": f"whole workload per step ({g.name})",
                             "host": host_cpu()},
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _timed(torch, flush, stream, fn, reps=5):
    """Median CUDA-event ms of fn() over reps calls (L2 flushed before each; one warm-up call
    first), last result.  The median keeps one slow outlier from moving the figure."""
    fn()
    ms, out = [], None
    for _ in range(reps):
        flush.fill_(3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = fn()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return sorted(ms)[len(ms) // 2], out


def clean_input_ms(tc, torch, rp, cl, flush, stream, T):
    """SURVEY §8(d)'s own definition of the headline ms: from a CLEAN symmetric CSR resident on
    the device (TC_CLEAN | TC_SORTED: a1 skipped) to the count.  The clean CSR is prepared
    outside the timed region from the library's oriented CSR (torch sort: input plumbing)."""
    crp, ccl = clean_csr_of(tc, torch, rp, cl)
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
    # pruning runs in the general pipeline: the unpruned reference is the pipeline's count
    bms, Tb = _timed(torch, flush, stream, lambda: tc.count_ex(rrp, rcl, lowdeg_max=0))
    sb = tc.count_ex(rrp, rcl, lowdeg_max=0, with_stats=True)[1]
    out = {"workload": g.name, "count_ms_unpruned": bms, "m": sb["m_undirected"],
           "note": "unpruned = the general pipeline (lowdeg_max = 0); the default bounded-degree "
                   "path counts this graph without pruning in other_configs"}
    for r in (1, 2, 0):
        pms, (Tp, sp) = _timed(torch, flush, stream,
                               lambda: tc.count_ex(rrp, rcl, prune=True, prune_rounds=r, with_stats=True))
        assert Tp == Tb
        out[f"rounds={r or 'fixed-point'}"] = {
            "ms_per_call": pms, "prune_ms": sp["ms_prune"], "pruned_edges": sp["pruned_edges"],
            "rounds_run": sp["prune_rounds"], "edges_per_s": sb["m_undirected"] / (pms * 1e-3)}
    rows["NEXT-2 leaf pruning (road mesh)"] = out
    return rows


def other_configs(tc, torch, np, graphgen, dev, flush, stream):
    """BASELINE configs[2] and [3] beside the headline (configs[1]): each graph's raw arcs
    resident on the device, one tc_count_ex per call (median of 5, L2 flushed), through the
    default path (the road mesh takes the bounded-degree path, DESIGN §4 step 8) and, for the
    road mesh, the general pipeline (lowdeg_max = 0) and the clean sorted CSR; plus the
    clique union (co-author-like).  Counts agree across paths (asserted); the parity tests hold
    them against the oracle."""
    rows = {}
    for name, make in (("road mesh (configs[3])", graphgen.road_mesh),
                       ("Chung-Lu LiveJournal-like (configs[2])", graphgen.chung_lu),
                       ("clique union (co-author-like)", graphgen.clique_union)):
        g = make()
        rp = torch.from_numpy(g.rowptr.view(np.int64)).to(dev)
        cl = torch.from_numpy(g.col.view(np.int32)).to(dev)
        ms, T = _timed(torch, flush, stream, lambda: tc.count_ex(rp, cl))
        T2, st = tc.count_ex(rp, cl, with_stats=True)   # (stats: untimed; they add work)
        assert T2 == T
        m = st["m_undirected"]
        row = {"workload": g.name, "n": g.n, "raw_arcs": g.arcs, "m": m, "T": T, "ms_per_call": ms,
               "edges_per_s": m / (ms * 1e-3), "launches": st["kernel_launches"]}
        if "road" in name:
            pms, Tp = _timed(torch, flush, stream, lambda: tc.count_ex(rp, cl, lowdeg_max=0))
            assert Tp == T
            sp = tc.count_ex(rp, cl, lowdeg_max=0, with_stats=True)[1]
            row["pipeline (lowdeg_max=0)"] = {"ms_per_call": pms, "launches": sp["kernel_launches"]}
            crp, ccl = clean_csr_of(tc, torch, rp, cl)
            cms, Tc = _timed(torch, flush, stream, lambda: tc.count_ex(crp, ccl, clean=True, sorted_rows=True))
            assert Tc == T
            row["clean sorted CSR"] = {"ms_per_call": cms, "edges_per_s": m / (cms * 1e-3)}
            del crp, ccl
        rows[name] = row
        del rp, cl
        torch.cuda.empty_cache()
    return rows


def small_graph_latency(tc, torch, graphgen, dev, reps=50):
    """Launch-bound regime: one synchronous tc_count_ex on Zachary's karate club
    (BASELINE configs[0]) from device pointers, host wall clock per call (median of `reps`),
    through the one-kernel small-graph path, the bounded-degree path and the general pipeline."""
    import numpy as np
    g = graphgen.karate()
    rp = torch.from_numpy(g.rowptr.view(np.int64)).to(dev)
    cl = torch.from_numpy(g.col.view(np.int32)).to(dev)
    out = {"workload": "karate (n=34, 78 edges)"}
    for name, kw in (("one_kernel", {}), ("bounded_degree", {"tiny_max_n": 0}),
                     ("pipeline", {"tiny_max_n": 0, "lowdeg_max": 0})):
        for _ in range(5):
            T, st = tc.count_ex(rp, cl, with_stats=True, **kw)
        us = []
        for _ in range(reps):
            t0 = time.perf_counter()
            T = tc.count_ex(rp, cl, **kw)
            us.append(1e6 * (time.perf_counter() - t0))
        assert T == 45
        out[name] = {"us_per_call": sorted(us)[len(us) // 2], "launches": st["kernel_launches"]}
    return out


# ------------------------------------------------------------------ a6 traffic (ncu, same run)
A6_KERNELS = "regex:k_hash|k_short|k_merge|k_search"
NCU_METRICS = ("dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
               "l1tex__throughput.avg.pct_of_peak_sustained_elapsed,"
               "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct")


def multi_gpu_projection(tc, torch, graphgen, np, rp, cl, one_gpu_ms, peak_gbs):
    """The sharded multi-GPU pipeline projected from ONE GPU (shard.emulate, timed: every rank's
    phases in turn with CUDA events, the collectives charged at the measured NVLink rates); the
    bench workload at worlds 2 / 4 / 8 and R-MAT s24 (BASELINE configs[4]) at world 8.  Context
    for the N > 1 runs, never a measured multi-GPU number."""
    from paper_1804_06926_b200 import shard

    def one(rp_, cl_, worlds, base_ms, b_a6):
        out = {}
        for w in worlds:
            shard.emulate(rp_, cl_, w)   # warm
            # best of 3 timed emulations: one emulated world holds every rank's buffers on this
            # GPU, and a run where the caching allocator has to map fresh memory mid-phase
            # (measured: a rank's count phase 34-38 ms instead of 7, a whole step 141 ms instead
            # of 18) says nothing about the ranks' kernels
            total, _, rep = min((shard.emulate(rp_, cl_, w, timed=True) for _ in range(3)),
                                key=lambda x: x[2]["step_ms_overlapped"])
            out[f"world{w}"] = {
                "T": total, "projected_step_ms": rep["step_ms_overlapped"],
                "speedup_vs_one_gpu": base_ms / rep["step_ms_overlapped"],
                "slowest_a6_ms": max(rep["a6_ms"]),
                "a6_aggregate_hbm_frac": b_a6 / (w * max(rep["a6_ms"]) * 1e-3) / (peak_gbs * 1e9),
                "phases_ms_slowest_rank": {k: max(v) for k, v in rep["phases"].items()},
                "collectives_ms": rep["collectives"]}
        return out

    _, st = tc.count_ex(rp, cl, with_stats=True)
    res = {"method": "one-GPU emulation (shard.emulate, best of 3 after a warm-up): each rank's phases "
                     "timed in turn with CUDA events; collectives charged at 770 GB/s (all-gather / all-to-all) and 725 GB/s "
                     "(all-reduce); the col+ all-gather overlapped with binning as run_rank does.  "
                     "NCCL was not run (one GPU per box this round)",
           "bench_workload": one(rp, cl, (2, 4, 8), one_gpu_ms, st["bytes_hash"] + st["bytes_core"])}
    g24 = graphgen.rmat(24, 16)
    rp24 = torch.from_numpy(g24.rowptr.view(np.int64)).to(rp.device)
    cl24 = torch.from_numpy(g24.col.view(np.int32)).to(rp.device)
    del g24
    for _ in range(2):
        _, st24 = tc.count_ex(rp24, cl24, with_stats=True)
    res["rmat-s24-ef16"] = {"one_gpu_ms": st24["ms_total"], **one(rp24, cl24, (8,), st24["ms_total"],
                                                                  st24["bytes_hash"] + st24["bytes_core"])}
    del rp24, cl24
    torch.cuda.empty_cache()
    return res


def clean_csr_of(tc, torch, rp, cl):
    """The symmetric, sorted, simple CSR of the graph (input plumbing for SURVEY §8(d)'s clean-
    input measurement, built outside any timed region from the library's oriented CSR)."""
    n = rp.numel() - 1
    off, colp = tc.orient(rp, cl)
    src = torch.repeat_interleave(torch.arange(n, device=rp.device), off[1:] - off[:-1])
    dst = colp.to(torch.int64)
    b = max(1, (n - 1).bit_length())
    keys, _ = torch.sort(torch.cat([(src << b) | dst, (dst << b) | src]))
    s2, d2 = keys >> b, keys & ((1 << b) - 1)
    crp = torch.zeros(n + 1, dtype=torch.int64, device=rp.device)
    crp[1:] = torch.cumsum(torch.bincount(s2, minlength=n), 0)
    return crp, d2.to(torch.int32).contiguous()


def one_call(args):
    """--one-call: ONE tc_count_ex on the bench workload (the process ncu profiles);
    --clean-input: on its clean sorted CSR (TC_CLEAN | TC_SORTED)."""
    import numpy as np
    import torch
    import graphgen
    import paper_1804_06926_b200 as tc
    g = graphgen.rmat(args.scale, args.edge_factor)
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
    cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    if args.clean_input:
        rp, cl = clean_csr_of(tc, torch, rp, cl)
        print("T", tc.count_ex(rp, cl, clean=True, sorted_rows=True), flush=True)
        return
    print("T", tc.count_ex(rp, cl), flush=True)


def ncu_traffic(args):
    """DRAM bytes of the a6 kernels of one step, captured by ncu in THIS bench run (a child
    process, after the timed region; no timing is taken from it).  Also the bitmap kernel's
    L1/shared-memory and DRAM throughput % (what bounds it) and its L2 hit rate."""
    import csv
    import io
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return {"error": "ncu not found"}
    cmd = [ncu, "--metrics", NCU_METRICS, "-k", A6_KERNELS, "--csv", "--print-units", "base",
           "--clock-control", "none", sys.executable, os.path.abspath(__file__), "--one-call",
           "--scale", str(args.scale), "--edge-factor", str(args.edge_factor)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    except (OSError, subprocess.SubprocessError) as e:
        return {"error": f"ncu failed: {e}"}
    rows = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    if not rows:
        return {"error": f"ncu produced no rows (rc {r.returncode}): {r.stderr[-300:]}"}
    per = {}
    for rec in csv.DictReader(io.StringIO("\n".join(rows))):
        key = (rec["ID"], rec["Kernel Name"])
        try:
            per.setdefault(key, {})[rec["Metric Name"]] = float(rec["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    dram = sum(v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0) for v in per.values())
    ns = sum(v.get("gpu__time_duration.sum", 0) for v in per.values())
    top = max(per.items(), key=lambda kv: kv[1].get("gpu__time_duration.sum", 0))
    tv = top[1]
    return {"dram_bytes": dram, "launches": len(per), "ncu_ms": ns * 1e-6,
            "top_kernel": top[0][1].split("(")[0],
            "top_l1tex_pct": tv.get("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
            "top_dram_pct": tv.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "top_l2_hit_pct": tv.get("lts__t_sector_hit_rate.pct"),
            "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (+ l1tex / dram "
                      f"throughput %, L2 hit rate) -k '{A6_KERNELS}' over one tc_count_ex of this "
                      "workload, run by this bench.py after its timed region (cold caches)"}


# ------------------------------------------------------------------ native arm
def main():
    args = parse()
    if args.one_call:
        return one_call(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_spawn(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import numpy as np
    import graphgen

    if args.impl == "reference" and rank != 0:
        return   # the reference arm (the CPU oracle) runs on rank 0 only
    g = graphgen.rmat(args.scale, args.edge_factor)
    if args.impl == "reference":
        line = reference_arm(args, g, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import torch
    import paper_1804_06926_b200 as tc
    from paper_1804_06926_b200.dist import (Comm, count_distributed, count_distributed_sharded,
                                            count_distributed_sharded_a1, exchange_clean_shards)
    from paper_1804_06926_b200.shard import run_rank
    # TC_BENCH_SHARED_GPU=1 (tests only): every rank on cuda:0 over gloo -- the boxes of this
    # round have one GPU and NCCL refuses two ranks on one device; the numbers are then
    # meaningless, the point is exercising the N > 1 code path end to end
    shared = os.environ.get("TC_BENCH_SHARED_GPU") == "1"
    # TC_BENCH_FORCE_DIST=1 (tests only): a one-rank job through the N > 1 path (process group,
    # NCCL collectives of dist.Comm on one GPU) -- the NCCL code path exercised on a 1-GPU box
    multi = world > 1 or os.environ.get("TC_BENCH_FORCE_DIST") == "1"
    gpu = 0 if shared else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    dist = None
    if multi:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    rp = torch.from_numpy(g.rowptr.view(np.int64)).to(dev)
    cl = torch.from_numpy(g.col.view(np.int32)).to(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    partial = torch.zeros(1, dtype=torch.int64, device=dev)
    mode = "single" if not multi else ("replicated" if args.replicated_a1 else
                                        ("sharded-a1" if args.sharded_a1_only else "sharded"))
    comm = Comm() if multi else None
    base_st = None
    if mode == "sharded":
        # the graph's byte model and sizes (B_a6, m, W: properties of the whole graph, the same
        # on every rank) from one single-GPU call outside the timed region
        base_st = tc.count_ex(rp, cl, with_stats=True)[1]

    def step(with_stats=False):
        if not multi:
            return tc.count_ex(rp, cl, with_stats=with_stats)
        if mode == "sharded":   # a1-a5 split over the ranks too (shard.py run_rank)
            times = {} if with_stats else None
            part, _ = run_rank(rp, cl, rank, world, comm, times=times)
            comm.all_reduce(part)
            T = int(part.item())
            if not with_stats:
                return T
            st = dict(base_st)
            st.update(ms_clean=times["clean"], ms_orient=times["orient"] + times["partition"] + times["rows"],
                      ms_sort=0.0, ms_bin=times["work"] + times["route"], ms_intersect=times["count"],
                      ms_total=sum(times.values()), ms_collectives=times["comm"])
            return T, st
        if args.replicated_a1:   # every rank cleans all arcs (SURVEY §8(e) as written)
            st = tc.count_shard(rp, cl, rank, world, partial, with_stats=with_stats)
        else:                    # the cleaning step split over the ranks (dist.py)
            edges, deg = exchange_clean_shards(rp, cl)
            st = tc.count_edges_shard(g.n, edges, deg, rank, world, partial, with_stats=with_stats)
        dist.all_reduce(partial)
        return (int(partial.item()), st) if with_stats else int(partial.item())

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, per-step CUDA events, L2 flushed between steps
    sampler = ClockSampler(gpu)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    stats = []
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    T_total = None
    launches0 = tc.launches_issued()
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        ev[k][0].record(stream)
        out = step(with_stats=True)
        ev[k][1].record(stream)
        T_total, st = out
        stats.append(st)
    torch.cuda.synchronize()
    launches = tc.launches_issued() - launches0   # this rank's kernels in the timed region
    if dist is not None:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / len(step_ms)
    ix_ms = sum(s["ms_intersect"] for s in stats) / len(stats)
    bin_ms = sum(s["ms_bin"] for s in stats) / len(stats)
    st = stats[-1]
    # per-rank work statistics (tc_stats counts this rank's edges): summed over ranks
    # a6 algorithmic bytes of the implemented method: HASH probes + ranges + table loads, plus
    # the dense-core path's word ANDs (8 bytes per word pair)
    b_hash, b_alg_rank = st["bytes_hash"] + st["bytes_core"], st["bytes_alg"]
    if dist is not None:
        t = torch.tensor([ms, ix_ms, bin_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ix_ms, bin_ms = t.tolist()
        # per-rank byte counts sum to the graph's; the sharded mode already has the whole graph's
        c = torch.tensor([b_hash if mode != "sharded" else 0, launches], dtype=torch.int64, device=dev)
        dist.all_reduce(c)
        if mode != "sharded":
            b_hash = int(c[0].item())
        launches = int(c[1].item())
    m = st["m_undirected"]

    # ---- end to end through the public API from pinned HOST buffers: every step copies the
    # raw CSR host->device, runs the whole path (N > 1: this rank's shard + the allreduce, via
    # count_distributed) and reads the count back; host wall clock, max over ranks
    e2e = None
    if not args.no_e2e:
        rp_h = torch.from_numpy(g.rowptr.view(np.int64)).pin_memory()
        cl_h = torch.from_numpy(g.col.view(np.int32)).pin_memory()

        def e2e_step():
            if not multi:
                return tc.count_ex(rp_h, cl_h, with_stats=True)[0]
            d_rp = rp_h.to(dev, non_blocking=True)
            d_cl = cl_h.to(dev, non_blocking=True)
            if mode == "replicated":
                return count_distributed(d_rp, d_cl)
            if mode == "sharded-a1":
                return count_distributed_sharded_a1(d_rp, d_cl)
            return count_distributed_sharded(d_rp, d_cl)

        e2e_step()   # warm
        reps = max(3, min(args.steps, 5))
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            got = e2e_step()
        e2e_s = (time.perf_counter() - t0) / reps
        assert got == T_total
        if dist is not None:
            t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = t.item()
        in_bytes = g.rowptr.nbytes + g.col.nbytes
        e2e = {"value": m / e2e_s, "unit": "edges/s", "ms_per_step": 1e3 * e2e_s,
               "h2d_bytes_per_step": in_bytes * world, "d2h_bytes_per_step": 8 * world,
               "note": ("tc_count_ex with TC_HOST_PTRS from pinned host memory" if not multi else
                        "count_distributed[_sharded[_a1]]: per rank H2D of the raw CSR (non_blocking "
                        "from pinned), the same path as the step, .item()") +
                       "; host wall clock per step, max over ranks"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    peak, peak_kind = load_peaks()
    b_alg = st["bytes_alg"] if world == 1 else None
    achieved = b_hash / (ix_ms * 1e-3) / 1e9 / world  # GB/s per GPU
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None,
            "kernel": "a6+a7 intersection phase (k_hash_cta bitmap + hash, k_hash_warp, k_short "
                      "[+ empty MERGE/SEARCH launches]), CUDA events on the launch stream",
            "bytes_model": "B_a6 = 4*(probes of HASH/SHORT edges) + 8*HASH edges + 4*table loads "
                           "+ 8*core words (bytes the implemented a6 must read; DESIGN.md sec. 5), "
                           "summed over ranks",
            "bytes_a6": b_hash, "bytes_core": st["bytes_core"], "core_edges": st["core_edges"],
            "kernel_ms": ix_ms, "bin_ms": bin_ms, "peak_kind": peak_kind,
            "work_W": st["work_W"], "work_probe": st["work_probe"], "table_loads": st["table_loads"]}
    if b_alg:
        a_alg = b_alg / (ix_ms * 1e-3) / 1e9
        roof["survey_B_alg"] = {"bytes": b_alg, "model": "4W + 16m (SURVEY.md 8(d), merge-based)",
                                "achieved": a_alg, "frac": a_alg / peak,
                                "frac_incl_binning": b_alg / ((ix_ms + bin_ms) * 1e-3) / 1e9 / peak}
        b_stage = 4 * (m + st["work_stage"]) + 16 * m
        roof["survey_B_stage"] = {"bytes": b_stage, "model": "4(m + sum d-(v) d+(v)) + 16m (SURVEY.md 8(d))",
                                  "frac": b_stage / (ix_ms * 1e-3) / 1e9 / peak}
    if not multi and not args.no_ncu:
        tr = ncu_traffic(args)
        roof["ncu"] = tr
        if "dram_bytes" in tr:
            roof["traffic"] = tr["dram_bytes"]
            roof["dram_frac"] = tr["dram_bytes"] / (ix_ms * 1e-3) / 1e9 / peak
            l1, dr = tr.get("top_l1tex_pct") or 0.0, tr.get("top_dram_pct") or 0.0
            # what ncu says binds the dominant kernel (report it, not "hbm")
            roof["bound"] = "l1/smem" if l1 > dr else "hbm"
            roof["bound_evidence"] = (f"{tr['top_kernel']}: L1TEX/shared {l1:.1f}% vs DRAM {dr:.1f}% "
                                      f"of peak, L2 hit {tr.get('top_l2_hit_pct') or 0:.1f}%")
    line = {
        "metric": METRIC, "value": m / (ms * 1e-3), "unit": "edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded R-MAT, Graph500 A,B,C,D=.57,.19,.19,.05; raw arcs)",
        "config": {"workload": g.name, "n": g.n, "m": m, "raw_arcs": g.arcs, "T": T_total,
                   "parallelism": (f"dp{world}: replicated input, owner-split intersection" +
                                   {"single": "", "replicated": ", a1-a5 replicated",
                                    "sharded-a1": ", sharded cleaning, a2-a5 replicated",
                                    "sharded": ", a1-a5 sharded (row-range CSR slices, all-gathered; "
                                               "HASH entries routed to their owner's rank)"}[mode]),
                   "l2": "flushed between timed steps (512 MiB write outside the event spans)",
                   "step": "tc_count_ex on raw arcs: clean, orient, bin, intersect, reduce"
                           + ({"single": "",
                               "replicated": " (tc_count_shard per rank) + NCCL allreduce",
                               "sharded-a1": " (tc_clean_shard per rank, NCCL all-reduce of degrees + "
                                             "all-gather of edges, tc_count_edges_shard, NCCL allreduce)",
                               "sharded": " (shard.py run_rank: tc_clean_shard / tc_shard_orient / "
                                          "partition / rows / work / route / count per rank between "
                                          "NCCL all-reduce, all-to-all and broadcast collectives, then "
                                          "the count all-reduce)"}[mode])},
        "phases_ms": {k: sum(s[k] for s in stats) / len(stats)
                      for k in ("ms_clean", "ms_orient", "ms_sort", "ms_bin", "ms_intersect", "ms_total")},
        "step_ms_min_max": [min(step_ms), max(step_ms)],
        "roofline": roof,
        "gpu_launches": launches,
        "e2e": e2e,
        "clocks": clocks,
    }
    if not multi and not args.no_next:
        # NEXT-1: clustering coefficients + transitivity on the same workload
        # through tc_clustering (count with t(v), then the c(v) kernel); median of 5 calls
        cms, (_, summ) = _timed(torch, flush, stream, lambda: tc.clustering(rp, cl))
        assert summ["triangles"] == T_total
        line["next_rows"] = {"NEXT-1 clustering": {
            "ms_per_call": cms, "edges_per_s": m / (cms * 1e-3), "overhead_vs_count_ms": cms - ms,
            "transitivity": summ["transitivity"], "avg_clustering": summ["avg_clustering"],
            "wedges": summ["wedges"], "timing": "median of 5 calls, L2 flushed before each",
            "call": "tc_clustering (device pointers): count with per-vertex t(v) + local c(v) for all n"}}
        line["survey_clean_input"] = clean_input_ms(tc, torch, rp, cl, flush, stream, T_total)
        line["small_graph"] = small_graph_latency(tc, torch, graphgen, dev)
        if not args.no_configs:
            line["other_configs"] = other_configs(tc, torch, np, graphgen, dev, flush, stream)
        line["next_rows"].update(next_rows_23(tc, torch, np, graphgen, rp, cl, flush, stream, m,
                                              T_total, ms))
    if not multi and not args.no_projection:
        line["multi_gpu_projection"] = multi_gpu_projection(tc, torch, graphgen, np, rp, cl, ms, peak)
    if not multi and not args.no_cpu_baseline:
        cb = cpu_baseline(g, m)
        assert cb.pop("T") == T_total, "oracle and CUDA path disagree"
        line["cpu_baseline"] = cb
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
