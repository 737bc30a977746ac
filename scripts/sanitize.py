"""Every entry point of the library on small graphs, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Exits non-zero on a wrong result."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import graphgen as G
import oracle as O
import paper_1804_06926_b200 as tc

graphs = [G.karate(), G.rmat(10, 16, seed=3), G.road_mesh(40, 30, seed=2),
          G.kron(G.karate(), G.fig_mm()), G.rmat(12, 16, seed=5)]   # s12: dense-core path
for g in graphs:
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    rp = torch.from_numpy(g.rowptr.view(np.int64)).cuda()
    cl = torch.from_numpy(g.col.view(np.int32)).cuda()
    for v in (None, tc.VARIANT_SHORT, tc.VARIANT_MERGE, tc.VARIANT_SEARCH, tc.VARIANT_HASH):
        got, pv = tc.count_ex(rp, cl, per_vertex=True, force_variant=v)
        assert got == T and (pv.cpu().numpy().view(np.uint64) == t).all(), (g.name, v)
    # the plain count through the pipeline (dense core) and through the one-kernel path
    assert tc.count_ex(rp, cl, tiny_max_n=0, lowdeg_max=0) == T and tc.count_ex(rp, cl) == T
    assert tc.count_ex(rp, cl, allocator="library") == T
    assert tc.count_ex(rp, cl, prune=True, hub_min_dplus=2) == T
    assert tc.count_ex(rp, cl, id_order=True) == T
    assert tc.clustering(rp, cl)[1]["triangles"] == T
    assert int(tc.edge_support(rp, cl)[2].to(torch.int64).sum().item()) == 3 * T
    assert tc.enumerate_triangles(rp, cl)[0] == T
    assert tc.masked_spgemm(rp, cl)[3] == T
    parts = []
    for r in range(3):
        p = torch.zeros(1, dtype=torch.int64, device="cuda")
        tc.count_shard(rp, cl, r, 3, p)
        parts.append(int(p.item()))
    assert sum(parts) == T
    # the sharded cleaning step (tc_clean_shard + tc_count_edges_shard), 2 ranks in turn
    cs = [tc.clean_shard(rp, cl, r, 2) for r in range(2)]
    edges = torch.cat([e for e, _ in cs])
    deg = (cs[0][1].to(torch.int64) + cs[1][1].to(torch.int64)).to(torch.int32)
    tot = 0
    for r in range(2):
        p = torch.zeros(1, dtype=torch.int64, device="cuda")
        tc.count_edges_shard(g.n, edges, deg, r, 2, p)
        tot += int(p.item())
    assert tot == T
    print(g.name, "ok", T, flush=True)
