"""Full-size parity of BASELINE configs[4] (R-MAT s24 ef16) on ONE GPU: the whole count and
the multi-GPU source split (tc_count_shard for world 2/4/8, every rank run on this GPU,
partials summed as the NCCL allreduce would) against the oracle on the host cores.
Writes one JSON line (committed under profiles/ as evidence; too slow for the default
pytest run: the oracle needs minutes at this size)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen as G
import oracle as O
import paper_1804_06926_b200 as tc

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
t0 = time.time()
g = G.rmat(scale, 16)
gen_s = time.time() - t0
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
cl = torch.from_numpy(g.col.view(np.int32)).cuda()
T_gpu, st = tc.count_ex(rp, cl, with_stats=True)
shards = {}
for world in (2, 4, 8):
    parts = []
    for r in range(world):
        p = torch.zeros(1, dtype=torch.int64, device="cuda")
        tc.count_shard(rp, cl, r, world, p)
        parts.append(int(p.item()))
    shards[world] = {"sum": sum(parts), "max_share": max(parts) / max(1, sum(parts)),
                     "partials": parts}
t1 = time.time()
T_or = O.count(g.n, g.rowptr, g.col)
or_s = time.time() - t1
ok = T_gpu == T_or and all(v["sum"] == T_or for v in shards.values())
print(json.dumps({"workload": g.name, "n": g.n, "raw_arcs": g.arcs, "m": st["m_undirected"],
                  "T_gpu": T_gpu, "T_oracle": T_or, "bit_exact": ok, "gpu_ms_total": st["ms_total"],
                  "gpu_ms_intersect": st["ms_intersect"], "shards": shards,
                  "oracle_s": or_s, "oracle_threads": O.num_threads(), "gen_s": gen_s}))
sys.exit(0 if ok else 1)
