"""Development aid: phase timings on the BASELINE configs (cuda:0)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import paper_1804_06926_b200 as tc
if os.environ.get("TC_LIB"):
    tc._LIB_PATH = os.environ["TC_LIB"]
which = sys.argv[1:] or ["s22", "s24", "chung_lu", "road", "clique"]
for w in which:
    t = time.time()
    g = {"s21": lambda: G.rmat(21), "s22": lambda: G.rmat(22), "s23": lambda: G.rmat(23),
         "s24": lambda: G.rmat(24), "chung_lu": G.chung_lu, "road": G.road_mesh,
         "clique": G.clique_union, "ef48": lambda: G.rmat(21, 48, seed=4821)}[w]()
    tg = time.time() - t
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda(); cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    for it in range(3):
        T, st = tc.count_ex(rp, cl, with_stats=True)
    frac = st["bytes_alg"] / (st["ms_intersect"] * 1e-3) / 6545.6e9
    print(f"{w}: gen {tg:.1f}s arcs={g.arcs} m={st['m_undirected']} T={T} total={st['ms_total']:.2f}ms "
          f"clean={st['ms_clean']:.2f} orient={st['ms_orient']:.2f} bin={st['ms_bin']:.2f} "
          f"ix={st['ms_intersect']:.2f} Balg/t={frac:.2f} edges/s={st['m_undirected']/st['ms_total']*1e3:.3e} "
          f"maxd+={st['max_dplus']} hubs={st['hub_sources']}", flush=True)
    del rp, cl
    torch.cuda.empty_cache()
