"""Development aid: one tc_clustering call on R-MAT sN (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 21
g = G.rmat(scale, 16)
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
cc, s = tc.clustering(rp, cl)
torch.cuda.synchronize()
print(s)
