"""Development aid: the bounded-degree path and the 16-bit in-part entries on small graphs, for
compute-sanitizer (memcheck / racecheck): dirty, clean sorted / unsorted, per-vertex, fallback."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as G
import oracle as O
import paper_1804_06926_b200 as tc
dev = torch.device("cuda:0")
def d(a, t):
    return torch.from_numpy(np.ascontiguousarray(a).view(t)).to(dev)
for g in (G.road_mesh(80, 60, seed=1), G.dirty(G.triangulated_grid(50, 40), seed=2),
          G.gnp(3000, 0.002, seed=3), G.from_edges(1600, [(0, i) for i in range(1, 40)] + [(1, 2), (2, 3), (1, 3)]),
          G.rmat(12, 16, seed=5)):
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    rp, cl = d(g.rowptr, np.int64), d(g.col, np.int32)
    got, pv = tc.count_ex(rp, cl, per_vertex=True, allocator="library")
    assert got == T and (pv.cpu().numpy().view(np.uint64) == t).all(), g.name
    row, col = O.clean(g.n, g.rowptr, g.col)
    assert tc.count_ex(d(row, np.int64), d(col, np.int32), clean=True, sorted_rows=True, allocator="library") == T
    assert tc.count_ex(d(row, np.int64), d(col, np.int32), clean=True, allocator="library") == T
    assert tc.count_ex(rp, cl, lowdeg_max=0, allocator="library") == T
    print(g.name, T, "ok", flush=True)
