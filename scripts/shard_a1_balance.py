"""Multi-GPU projection with the cleaning step sharded (tc_clean_shard + exchange +
tc_count_edges_shard), emulated on ONE GPU: every rank's calls run in turn (CUDA events),
the exchange is done locally and charged at the measured NVLink figures of
B200_PROFILING.md (all-gather 770 GB/s per direction per GPU, all-reduce bus 725 GB/s).
The slowest rank's clean + exchange + count bounds the N-GPU step."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen as G
import paper_1804_06926_b200 as tc

if os.environ.get("TC_LIB"):
    tc._LIB_PATH = os.environ["TC_LIB"]


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b), out


for scale in [int(x) for x in sys.argv[1:]] or [21, 24]:
    g = G.rmat(scale, 16)
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
    cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    T1, st1 = tc.count_ex(rp, cl, with_stats=True)
    T1, st1 = tc.count_ex(rp, cl, with_stats=True)
    res = {"T": T1, "world1_total_ms": st1["ms_total"]}
    for world in (2, 4, 8):
        tc.clean_shard(rp, cl, 0, world)   # warm
        cleans, parts = [], []
        for r in range(world):
            ms, (e, d) = timed(lambda: tc.clean_shard(rp, cl, r, world))
            cleans.append(ms)
            parts.append((e.clone(), d.clone()))
        edges = torch.cat([e for e, _ in parts])
        deg = sum(d.to(torch.int64) for _, d in parts).to(torch.int32)
        del parts
        m_max = max(int(edges.numel() / world * 1.2), 1)
        gather_ms = 8.0 * edges.numel() * (world - 1) / world / 770e9 * 1e3
        allreduce_ms = 4.0 * g.n * 2 * (world - 1) / world / 725e9 * 1e3
        counts, tot = [], 0
        for r in range(world):
            p = torch.zeros(1, dtype=torch.int64, device="cuda")
            tc.count_edges_shard(g.n, edges, deg, r, world, p)   # warm
            ms, _ = timed(lambda: tc.count_edges_shard(g.n, edges, deg, r, world, p))
            counts.append(ms)
            tot += int(p.item())
        assert tot == T1
        steps = [c + gather_ms + allreduce_ms + k for c, k in zip(cleans, counts)]
        res[f"world{world}"] = {"clean_ms": cleans, "count_ms": counts, "exchange_ms": gather_ms + allreduce_ms,
                                "projected_step_ms": max(steps), "speedup_vs_world1": st1["ms_total"] / max(steps)}
        del edges, deg
        torch.cuda.empty_cache()
    print(json.dumps({g.name: res}), flush=True)
