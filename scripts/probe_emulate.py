"""Development aid: shard.emulate timed on R-MAT s24 at world 8 (per-rank phase ms)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
if os.environ.get("TC_LIB"):
    tc._LIB_PATH = os.environ["TC_LIB"]
from paper_1804_06926_b200 import shard
scale, world = int(sys.argv[1]), int(sys.argv[2])
g = G.rmat(scale, 16)
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
for it in range(2):
    total, _, rep = shard.emulate(rp, cl, world, timed=True)
    print(it, total, "step", round(rep["step_ms_overlapped"], 2), {k: [round(x, 2) for x in v] for k, v in rep["phases"].items() if k == "count"},
          "a6", [round(x, 2) for x in rep["a6_ms"]], "mem GB", round(torch.cuda.max_memory_reserved() / 1e9, 1), flush=True)
