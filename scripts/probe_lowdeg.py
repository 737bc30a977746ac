"""Development aid: the bounded-degree path (lowdeg.cu) against the general pipeline on the
road mesh (BASELINE configs[3]) -- dirty and clean-sorted input, median of 7 synchronous
calls (CUDA events around each), phase times from stats."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import oracle as O
import paper_1804_06926_b200 as tc
if os.environ.get("TC_LIB"):
    tc._LIB_PATH = os.environ["TC_LIB"]


def timed(rp, cl, **kw):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts, T = [], None
    for it in range(9):
        torch.cuda.synchronize()
        ev[0].record()
        T = tc.count_ex(rp, cl, **kw)
        ev[1].record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(ev[0].elapsed_time(ev[1]))
    _, st = tc.count_ex(rp, cl, with_stats=True, **kw)
    return T, statistics.median(ts), st


which = sys.argv[1:] or ["road"]
for w in which:
    g = {"road": G.road_mesh, "road_small": lambda: G.road_mesh(1000, 1000),
         "tri": lambda: G.triangulated_grid(3753, 3753)}[w]()
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
    cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    row, col = O.clean(g.n, g.rowptr, g.col)
    rpc = torch.from_numpy(row.view(np.int64)).cuda()
    clc = torch.from_numpy(col.view(np.int32)).cuda()
    for label, (a, b), kw in [("dirty lowdeg", (rp, cl), {}), ("dirty pipeline", (rp, cl), {"lowdeg_max": 0}),
                              ("clean lowdeg", (rpc, clc), {"clean": True, "sorted_rows": True}),
                              ("clean pipeline", (rpc, clc), {"clean": True, "sorted_rows": True, "lowdeg_max": 0})]:
        T, ms, st = timed(a, b, **kw)
        print(f"{os.environ.get('TC_LIB', '')} {w} {label}: T={T} m={st['m_undirected']} call {ms:.3f} ms (stats call: total "
              f"{st['ms_total']:.3f} clean {st['ms_clean']:.3f} orient {st['ms_orient']:.3f} bin "
              f"{st['ms_bin']:.3f} ix {st['ms_intersect']:.3f}) launches {st['kernel_launches']} "
              f"edges/s {st['m_undirected'] / ms * 1e3:.3e}", flush=True)
