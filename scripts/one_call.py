"""Development aid: one tc_count_ex call on R-MAT sN (for ncu launch lists)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 21
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
g = G.rmat(scale, 16)
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
T, st = tc.count_ex(rp, cl, with_stats=True, **kw)
print("T", T, {k: st[k] for k in ("ms_total", "ms_intersect", "kernel_launches", "hub_sources")})
