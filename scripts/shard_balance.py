"""Multi-GPU load balance evidence on ONE GPU: every rank's share (tc_count_shard) of the
same graph run one after another, with its intersection-phase time.  The slowest rank
bounds an N-GPU step; max/mean of the a6+a7 times measures the source split."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen as G
import paper_1804_06926_b200 as tc

if os.environ.get("TC_LIB"):   # a variants/<name>/libtc_b200.so build
    tc._LIB_PATH = os.environ["TC_LIB"]

out = {}
for scale in [int(a) for a in sys.argv[1:]] or [21, 24]:
    g = G.rmat(scale, 16)
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
    cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    T1, st1 = tc.count_ex(rp, cl, with_stats=True)
    T1, st1 = tc.count_ex(rp, cl, with_stats=True)
    res = {"T": T1, "ix_ms_world1": st1["ms_intersect"], "total_ms_world1": st1["ms_total"]}
    for world in (2, 4, 8):
        ix, tot, parts = [], [], []
        for r in range(world):
            p = torch.zeros(1, dtype=torch.int64, device="cuda")
            tc.count_shard(rp, cl, r, world, p)                     # warm
            st = tc.count_shard(rp, cl, r, world, p, with_stats=True)
            ix.append(st["ms_intersect"])
            tot.append(st["ms_total"])
            parts.append(int(p.item()))
        assert sum(parts) == T1
        res[f"world{world}"] = {"ix_ms": ix, "ix_max_over_mean": max(ix) / (sum(ix) / world),
                                "ix_speedup": st1["ms_intersect"] / max(ix),
                                "ix_sum_over_world1": sum(ix) / st1["ms_intersect"],
                                "total_ms_per_rank": tot, "projected_step_ms": max(tot)}
    out[g.name] = res
    print(json.dumps({g.name: res}), flush=True)
    del rp, cl
    torch.cuda.empty_cache()
