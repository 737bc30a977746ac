"""Multi-GPU projection of the SHARDED pipeline (shard.py / csrc/shard.cu): every rank of a
world run in turn on ONE B200 (shard.emulate, timed=True: each phase of each rank bracketed by
CUDA events), the collectives charged at the measured NVLink figures of B200_PROFILING.md.
Projected step = sum over phases of the slowest rank + the collectives.  Also the a6 phase's
aggregate HBM roofline fraction: B_a6 of the whole graph (bench.py's byte model, from the
one-GPU stats) / (world x slowest count phase x peak)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen as G
import paper_1804_06926_b200 as tc
from paper_1804_06926_b200 import shard

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
out = {}
for scale in [int(x) for x in sys.argv[1:]] or [21, 24]:
    g = G.rmat(scale, 16)
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
    cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    for _ in range(2):
        T1, st = tc.count_ex(rp, cl, with_stats=True)
    b_a6 = st["bytes_hash"] + st["bytes_core"]   # bench.py's B_a6
    res = {"T": T1, "world1_total_ms": st["ms_total"], "world1_a6_ms": st["ms_intersect"]}
    for world in (1, 2, 4, 8):
        shard.emulate(rp, cl, world)   # warm
        total, _, rep = shard.emulate(rp, cl, world, timed=True)
        assert total == T1, (scale, world, total, T1)
        cnt = max(rep["phases"]["count"])
        rep["count_phase_aggregate_hbm_frac"] = b_a6 / (world * cnt * 1e-3) / PEAK
        # the intersection phase proper (north_star: "at >= 50% of aggregate HBM roofline for
        # the intersection phase"): the slowest rank's a6 + a7 kernel span
        rep["a6_aggregate_hbm_frac"] = b_a6 / (world * max(rep["a6_ms"]) * 1e-3) / PEAK
        rep["speedup_vs_world1"] = st["ms_total"] / rep["step_ms"]
        res[f"world{world}"] = rep
        print(scale, world, "step", round(rep["step_ms"], 2), "ms",
              {k: round(max(v), 2) for k, v in rep["phases"].items()},
              {k: round(v, 2) for k, v in rep["collectives"].items()}, flush=True)
    out[f"rmat-s{scale}-ef16"] = res
print(json.dumps(out))
