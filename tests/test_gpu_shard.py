"""GPU parity of the sharded multi-GPU pipeline (csrc/shard.cu, shard.py): every
rank of a world run in turn on ONE GPU (shard.emulate: the collectives are local tensor
operations), and the ranks' partial counts / per-vertex partials must sum to the oracle's T and
t(v) bit for bit (Alg. 2), for several worlds, graphs, the per-vertex mode (no dense
core) and the dense-core count mode.  The gathered oriented CSR must equal the oracle's
orientation (rank order (d, id))."""
import numpy as np
import pytest

import graphgen as G
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1804_06926_b200 import shard  # noqa: E402

DEV = torch.device("cuda:0")


def on_dev(g):
    return (torch.from_numpy(np.ascontiguousarray(g.rowptr, np.uint64).view(np.int64)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(g.col, np.uint32).view(np.int32)).to(DEV))


GRAPHS = {
    "karate": G.karate,
    "rmat12": lambda: G.rmat(12, 16, seed=21),
    "rmat15_dirty": lambda: G.dirty(G.rmat(15, 8, seed=15), 15),
    "chung_lu": lambda: G.chung_lu(30000, 300000, seed=6),
    "clique": lambda: G.clique_union(30000, 40000, seed=2),
    "mesh": lambda: G.road_mesh(300, 200, seed=3),
    "star": lambda: G.star(5000),
}


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_sharded_count(name, world):
    g = GRAPHS[name]()
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    rp, cl = on_dev(g)
    total, _, _ = shard.emulate(rp, cl, world)
    assert total == T, (name, world, total, T)
    total, pv, _ = shard.emulate(rp, cl, world, per_vertex=True)
    assert total == T and (pv.cpu().numpy().view(np.uint64) == t).all(), (name, world)


@pytest.mark.parametrize("world", [2, 5])
def test_sharded_policy_knobs(world):
    g = G.rmat(13, 16, seed=4)
    T = O.count(g.n, g.rowptr, g.col)
    rp, cl = on_dev(g)
    for kw in [dict(short_max=0), dict(short_max=64), dict(hub_min_dplus=2), dict(skew_ratio=4),
               dict(hub_min_dplus=1 << 20)]:
        total, _, _ = shard.emulate(rp, cl, world, **kw)
        assert total == T, kw


def test_sharded_csr_equals_oracle():
    """The gathered col+ (rank ids) mapped back to input ids is the oracle's oriented CSR."""
    g = G.dirty(G.rmat(12, 16, seed=8), 8)
    rp, cl = on_dev(g)
    n, world = g.n, 4
    row, col = O.clean(g.n, g.rowptr, g.col)
    want_off, want_col = O.orient(g.n, row, col)
    cls = [shard.clean_shard(rp, cl, r, world) for r in range(world)]
    deg = sum(d.to(torch.int64) for _, d in cls).to(torch.int32)
    p1 = [shard.shard_orient(n, e, deg) for e, _ in cls]
    dplus = sum(p[3].to(torch.int64) for p in p1).to(torch.int32)
    p2 = [shard.shard_partition(n, p[1], p[2], dplus, r, world) for r, p in enumerate(p1)]
    off, cb = p2[0][0], p2[0][4]
    col_plus = torch.empty(cb[world], dtype=torch.int32, device=DEV)
    for q in range(world):
        parts = []
        for r in range(world):
            c = p2[r][2]
            parts.append(p2[r][1][sum(c[:q]):sum(c[:q]) + c[q]])
        shard.shard_rows(n, torch.cat(parts), col_plus, cb[q])
    newid = p1[0][0].cpu().numpy().astype(np.int64)
    order = np.empty(n, np.int64)
    order[newid] = np.arange(n)
    offn, coln = off.cpu().numpy(), col_plus.cpu().numpy().astype(np.int64)
    # row x of the rank-id CSR = N+(order[x]); in input ids each row is a set: compare sorted
    got = {}
    for x in range(n):
        a, b = offn[x], offn[x + 1]
        if b > a:
            got[int(order[x])] = np.sort(order[coln[a:b]])
    wo = want_off.astype(np.int64)
    for v in range(n):
        w = np.sort(want_col[wo[v]:wo[v + 1]].astype(np.int64))
        assert np.array_equal(got.get(v, np.zeros(0, np.int64)), w), v
