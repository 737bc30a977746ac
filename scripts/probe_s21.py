"""Development aid: phase timings of the pipeline on R-MAT sN (cuda:0) under several policies."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
if os.environ.get("TC_LIB"):
    tc._LIB_PATH = os.environ["TC_LIB"]
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 21
t = time.time(); g = G.rmat(scale, 16); print("gen", round(time.time() - t, 2), "s arcs", g.arcs, flush=True)
rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
import json
cfgs = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [dict(force_variant=v) for v in [0, 1, 2, 3]] + [{}]
for kw in cfgs:
    for it in range(3):
        T, st = tc.count_ex(rp, cl, with_stats=True, **kw)
    print(f"{kw}: T={T} total={st['ms_total']:.2f}ms clean={st['ms_clean']:.2f} orient={st['ms_orient']:.2f} "
          f"bin={st['ms_bin']:.2f} ix={st['ms_intersect']:.2f} bins={st['bin_edges']} hubs={st['hub_sources']} "
          f"probe={st['work_probe']:.3e} W={st['work_W']:.3e}", flush=True)
