"""Largest config of BASELINE (R-MAT s25/s26 ef16) on one GPU, no oracle (it would take
hours): the whole count, and the sum of the 8 shards of the multi-GPU split (each run on
this GPU) must agree; per-phase times and peak device memory."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
t0 = time.time()
g = G.rmat(scale, 16)
gen = time.time() - t0
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
cl = torch.from_numpy(g.col.view(np.int32)).cuda()
torch.cuda.reset_peak_memory_stats()
free0, tot = torch.cuda.mem_get_info()
T, st = tc.count_ex(rp, cl, with_stats=True)
T, st = tc.count_ex(rp, cl, with_stats=True)
parts = []
for r in range(8):
    p = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.count_shard(rp, cl, r, 8, p)
    parts.append(int(p.item()))
free1, _ = torch.cuda.mem_get_info()
ok = sum(parts) == T
print(json.dumps({"workload": g.name, "raw_arcs": g.arcs, "m": st["m_undirected"], "T": T,
                  "shards8_sum_equal": ok, "ms_total": st["ms_total"],
                  "phases_ms": {k: st[k] for k in ("ms_clean", "ms_orient", "ms_bin", "ms_intersect")},
                  "max_dplus": st["max_dplus"], "gen_s": gen,
                  "device_free_gb_before_after": [free0 / 1e9, free1 / 1e9]}))
sys.exit(0 if ok else 1)
