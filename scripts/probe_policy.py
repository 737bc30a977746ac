"""Development aid: AUTO-policy sweep on several configs."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
mk = {"s21": lambda: G.rmat(21), "chung_lu": G.chung_lu, "road": G.road_mesh, "clique": G.clique_union,
      "s24": lambda: G.rmat(24), "s22": lambda: G.rmat(22), "ef48": lambda: G.rmat(21, 48)}
cfgs = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [{}]
for w in sys.argv[1].split(","):
    g = mk[w]()
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    for kw in cfgs:
        for _ in range(3):
            T, st = tc.count_ex(rp, cl, with_stats=True, **kw)
        print(f"{w} {kw}: total={st['ms_total']:.2f} orient={st['ms_orient']:.2f} bin={st['ms_bin']:.2f} ix={st['ms_intersect']:.2f} bins={st['bin_edges']}", flush=True)
    del rp, cl; torch.cuda.empty_cache()
