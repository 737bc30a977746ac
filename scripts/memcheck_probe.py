"""Development aid: one library call per argv case, for compute-sanitizer triage."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
case = sys.argv[1]
g = {"karate": G.karate, "rmat10": lambda: G.rmat(10, 16, seed=3), "k20": lambda: G.complete(20),
     "mesh": lambda: G.road_mesh(40, 30, seed=2)}[sys.argv[2]]()
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
kw = {"pv": dict(per_vertex=True), "count": dict(), "pv_hash": dict(per_vertex=True, force_variant=3),
      "count_hash": dict(force_variant=3), "pv_hub2": dict(per_vertex=True, hub_min_dplus=2)}[case]
print(case, sys.argv[2], tc.count_ex(rp, cl, **kw) if "pv" not in case else tc.count_ex(rp, cl, **kw)[0])
