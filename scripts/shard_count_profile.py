"""Development aid: one emulated world's count phase of one rank under ncu
(TC_PROFILE_COUNT_RANK; run with ncu --profile-from-start off)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
from paper_1804_06926_b200 import shard
scale, world = int(sys.argv[1]), int(sys.argv[2])
g = G.rmat(scale, 16)
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
print(shard.emulate(rp, cl, world)[0])
