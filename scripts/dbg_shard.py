import sys, torch, numpy as np
sys.path.insert(0, '.')
import graphgen as G, oracle as O, paper_1804_06926_b200 as tc
g = G.rmat(12, 16, seed=21)
T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
rp = torch.from_numpy(g.rowptr.astype(np.int64)).cuda(); cl = torch.from_numpy(g.col.astype(np.int32)).cuda()
for kw in [dict(), dict(short_max=0), dict(short_max=4), dict(force_variant=0)]:
    for world in [1, 2, 3, 8]:
        parts = []
        pvs = torch.zeros(g.n, dtype=torch.int64, device='cuda')
        for r in range(world):
            partial = torch.zeros(1, dtype=torch.int64, device='cuda')
            pv = torch.zeros(g.n, dtype=torch.int64, device='cuda')
            tc.count_shard(rp, cl, r, world, partial, per_vertex_partial=pv, **kw)
            torch.cuda.synchronize(); parts.append(int(partial.item())); pvs += pv
        print(kw, world, T, sum(parts), parts, int((pvs.cpu().numpy() != t.astype(np.int64)).sum()))
