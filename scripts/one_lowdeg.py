"""Development aid: one bounded-degree call on the road mesh (dirty, then clean sorted), for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import oracle as O
import paper_1804_06926_b200 as tc
if os.environ.get("TC_LIB"):
    tc._LIB_PATH = os.environ["TC_LIB"]
g = G.road_mesh()
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
cl = torch.from_numpy(g.col.view(np.int32)).cuda()
print(tc.count_ex(rp, cl))
row, col = O.clean(g.n, g.rowptr, g.col)
print(tc.count_ex(torch.from_numpy(row.view(np.int64)).cuda(), torch.from_numpy(col.view(np.int32)).cuda(),
                  clean=True, sorted_rows=True))
