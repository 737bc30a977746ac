"""Development aid: one tc_count_ex call on a named config (for ncu)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
name = sys.argv[1]
g = G.rmat(int(name[4:]), 16) if name.startswith("rmat") else \
    {"road": G.road_mesh, "chung_lu": G.chung_lu, "clique": G.clique_union, "karate": G.karate}[name]()
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
reps = int(os.environ.get("REPS", "1"))
for _ in range(reps):
    T, st = tc.count_ex(rp, cl, with_stats=True, **kw)
print("T", T, st["ms_total"])
