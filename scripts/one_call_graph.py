"""Development aid: one tc_count_ex call on a named config (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
g = {"road": G.road_mesh, "cl": G.chung_lu, "clique": G.clique_union}[sys.argv[1]]()
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
T, st = tc.count_ex(rp, cl, with_stats=True)
print("T", T, {k: st[k] for k in ("ms_total", "ms_clean", "ms_orient", "ms_bin", "ms_intersect")})
