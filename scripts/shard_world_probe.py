"""Development aid: one emulated world (timed) for library variants: TC_LIBS=a:path,..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
from paper_1804_06926_b200 import shard
scale, world = int(sys.argv[1]), int(sys.argv[2])
g = G.rmat(scale, 16)
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
libs = [x.split(":", 1) for x in os.environ.get("TC_LIBS", "").split(",") if x] or [("tree", tc._LIB_PATH)]
for name, path in libs:
    tc._lib = None; tc._LIB_PATH = path; shard._SIG = False
    shard.emulate(rp, cl, world)
    T, _, rep = shard.emulate(rp, cl, world, timed=True)
    print(name, T, "step", round(rep["step_ms"], 2), "a6", [round(x, 2) for x in rep["a6_ms"]],
          "count", [round(x, 2) for x in rep["phases"]["count"]], flush=True)
