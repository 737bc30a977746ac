"""GPU parity of the NEXT rows through the C ABI against the oracle.

NEXT-2 (TC_PRUNE leaf pruning): the oriented CSR of the pruned graph element by
element, T and every t(v) bit-exact, the pruned-edge and round counts.
"""
import numpy as np
import pytest

import graphgen as G
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1804_06926_b200 as tc  # noqa: E402

DEV = torch.device("cuda:0")
VARIANTS = [None, tc.VARIANT_SHORT, tc.VARIANT_MERGE, tc.VARIANT_SEARCH, tc.VARIANT_HASH]


def on_dev(rowptr, col):
    return (torch.from_numpy(np.ascontiguousarray(rowptr, np.uint64).view(np.int64)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(col, np.uint32).view(np.int32)).to(DEV))


def lollipop(L):
    e = [(i, j) for i in range(5) for j in range(i + 1, 5)] + [(4 + i, 5 + i) for i in range(L)]
    return G.from_edges(5 + L, e, f"lollipop{L}")


PRUNE_GRAPHS = {
    "lollipop9": lambda: lollipop(9),
    "path40": lambda: G.path(40),
    "tree": lambda: G.random_tree(3000, 2),
    "mesh": lambda: G.road_mesh(120, 90, seed=6),
    "rmat12": lambda: G.rmat(12, 4, seed=2),
    "gnp": lambda: G.gnp(3000, 0.0007, 3),
    "dirty_karate": lambda: G.dirty(G.karate(), seed=1),
}


def oracle_pruned(g, rounds):
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    prow, pcol, done = O.prune(g.n, crow, ccol, rounds)
    off, colp = O.orient(g.n, prow, pcol)
    return (int(crow[g.n]) - int(prow[g.n])) // 2, done, off, colp, crow, ccol


@pytest.mark.parametrize("name", list(PRUNE_GRAPHS))
@pytest.mark.parametrize("rounds", [0, 1, 2, 5])
def test_prune_orientation_parity(name, rounds):
    g = PRUNE_GRAPHS[name]()
    pruned, done, want_off, want_col, crow, ccol = oracle_pruned(g, rounds)
    for clean in (False, True):
        rp, cl = on_dev(crow, ccol) if clean else on_dev(g.rowptr, g.col)
        off, colp = tc.orient(rp, cl, clean=clean, sorted_rows=clean, prune=True, prune_rounds=rounds)
        torch.cuda.synchronize()
        assert (off.cpu().numpy().view(np.uint64) == want_off).all(), (name, rounds, clean)
        assert (colp.cpu().numpy().view(np.uint32) == want_col).all(), (name, rounds, clean)
        T, st = tc.count_ex(rp, cl, clean=clean, sorted_rows=clean, prune=True, prune_rounds=rounds,
                            with_stats=True)
        assert st["pruned_edges"] == pruned and st["prune_rounds"] == done, (name, rounds, clean)
        assert st["m_undirected"] == len(want_col)


@pytest.mark.parametrize("name", ["mesh", "rmat12", "dirty_karate", "lollipop9"])
def test_prune_counts_all_variants(name):
    g = PRUNE_GRAPHS[name]()
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    for v in VARIANTS:
        for rounds in (0, 1, 3):
            rp, cl = on_dev(g.rowptr, g.col)
            got, pv = tc.count_ex(rp, cl, per_vertex=True, prune=True, prune_rounds=rounds,
                                  force_variant=v)
            torch.cuda.synchronize()
            assert got == T and (pv.cpu().numpy().view(np.uint64) == t).all(), (name, v, rounds)


def test_prune_host_pointers_and_shards():
    g = G.road_mesh(150, 150, seed=9)
    T = O.count(g.n, g.rowptr, g.col)
    assert tc.count_ex(g.rowptr, g.col, prune=True) == T          # TC_HOST_PTRS path
    rp, cl = on_dev(g.rowptr, g.col)
    parts = []
    for r in range(3):
        p = torch.zeros(1, dtype=torch.int64, device=DEV)
        tc.count_shard(rp, cl, r, 3, p, prune=True, prune_rounds=2)
        parts.append(int(p.item()))
    assert sum(parts) == T


def test_prune_everything_and_degenerate():
    for g in (G.random_tree(500, 7), G.star(50), G.path(2), G.from_edges(5, [])):
        rp, cl = on_dev(g.rowptr, g.col)
        T, st = tc.count_ex(rp, cl, prune=True, with_stats=True)
        assert T == 0
        off, colp = tc.orient(rp, cl, prune=True)
        assert len(colp) == 0 and int(off[-1].item()) == 0


def test_prune_config_road_full():
    """BASELINE configs[3] (road mesh, the filter-dominated regime) under 2-core pruning."""
    g = G.road_mesh()
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    pruned, done, want_off, want_col, _, _ = oracle_pruned(g, 0)
    rp, cl = on_dev(g.rowptr, g.col)
    got, pv, st = tc.count_ex(rp, cl, per_vertex=True, prune=True, with_stats=True)
    assert got == T and (pv.cpu().numpy().view(np.uint64) == t).all()
    assert st["pruned_edges"] == pruned and st["prune_rounds"] == done
    off, colp = tc.orient(rp, cl, prune=True)
    assert (off.cpu().numpy().view(np.uint64) == want_off).all()
    assert (colp.cpu().numpy().view(np.uint32) == want_col).all()


# ------------------------------------------------------------------ NEXT-3: edge support
SUPPORT_GRAPHS = {
    "fig_mm": G.fig_mm,
    "karate": G.karate,
    "K40": lambda: G.complete(40),
    "wheel30": lambda: G.wheel(30),
    "rmat12_dirty": lambda: G.rmat(12, 16, seed=3),
    "gnp": lambda: G.gnp(600, 0.04, 5),
    "cliques": lambda: G.clique_union(6000, 5000, seed=4),
    "mesh": lambda: G.road_mesh(100, 80, seed=2),
    "kron": lambda: G.kron(G.karate(), G.fig_mm()),
}


def oracle_support(g):
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    off, colp = O.orient(g.n, crow, ccol)
    return off, colp, O.edge_support(g.n, crow, ccol, off, colp)


def np_u(t, dt):
    return t.cpu().numpy().view(dt) if hasattr(t, "cpu") else np.asarray(t).view(dt)


@pytest.mark.parametrize("name", list(SUPPORT_GRAPHS))
def test_edge_support_parity(name):
    g = SUPPORT_GRAPHS[name]()
    want_off, want_col, want_sup = oracle_support(g)
    T = O.count(g.n, g.rowptr, g.col)
    for v in VARIANTS:
        rp, cl = on_dev(g.rowptr, g.col)
        off, colp, sup = tc.edge_support(rp, cl, force_variant=v)
        torch.cuda.synchronize()
        assert (np_u(off, np.uint64) == want_off).all() and (np_u(colp, np.uint32) == want_col).all()
        assert (np_u(sup, np.uint32) == want_sup).all(), (name, v)
    assert int(want_sup.sum()) == 3 * T


def test_edge_support_clean_host_prune_and_hubs():
    g = G.rmat(14, 16, seed=8)                       # CTA hash / bitmap owners
    want_off, want_col, want_sup = oracle_support(g)
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    for kw in (dict(), dict(hub_min_dplus=8), dict(short_max=0), dict(short_max=64)):
        off, colp, sup = tc.edge_support(g.rowptr, g.col, **kw)          # host pointers
        assert (off == want_off).all() and (colp == want_col).all() and (sup == want_sup).all(), kw
    rp, cl = on_dev(crow, ccol)
    off, colp, sup = tc.edge_support(rp, cl, clean=True, sorted_rows=True)
    assert (np_u(sup, np.uint32) == want_sup).all()
    # pruned: the same supports on the surviving (2-core) edges
    prow, pcol, _ = O.prune(g.n, crow, ccol, 0)
    poff, pcolp = O.orient(g.n, prow, pcol)
    psup = O.edge_support(g.n, prow, pcol, poff, pcolp)
    off, colp, sup = tc.edge_support(rp, cl, clean=True, sorted_rows=True, prune=True)
    assert (np_u(colp, np.uint32) == pcolp).all() and (np_u(sup, np.uint32) == psup).all()


def test_edge_support_degenerate():
    for g in (G.from_edges(0, []), G.from_edges(4, []), G.path(5), G.complete(3)):
        off, colp, sup = tc.edge_support(g.rowptr, g.col)
        want_off, want_col, want_sup = oracle_support(g)
        assert (off == want_off).all() and (sup == want_sup).all()


def test_edge_support_rmat21_full():
    """The bench workload (configs[1]): sum = 3T and sampled supports by definition."""
    g = G.rmat(21, 16)
    T = O.count(g.n, g.rowptr, g.col)
    rp, cl = on_dev(g.rowptr, g.col)
    off, colp, sup = tc.edge_support(rp, cl)
    off, colp, sup = np_u(off, np.uint64), np_u(colp, np.uint32), np_u(sup, np.uint32)
    assert int(sup.sum(dtype=np.uint64)) == 3 * T
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(off.astype(np.int64)))
    rng = np.random.default_rng(1)
    deg = np.diff(crow.astype(np.int64))
    hubs = np.argsort(deg)[-5:]
    hub_edges = np.nonzero(np.isin(src, hubs))[0][:300]
    for e in np.concatenate([rng.integers(0, len(colp), 700), hub_edges]):
        u, v = int(src[e]), int(colp[e])
        nu, nv = ccol[crow[u]:crow[u + 1]], ccol[crow[v]:crow[v + 1]]
        assert int(sup[e]) == np.intersect1d(nu, nv, assume_unique=True).size, (u, v)


# ------------------------------------------------------------------ NEXT-3: enumeration
def sorted_rows(tri):
    t = np.asarray(tri, dtype=np.int64)
    return t[np.lexsort((t[:, 2], t[:, 1], t[:, 0]))] if len(t) else t.reshape(0, 3)


@pytest.mark.parametrize("name", list(SUPPORT_GRAPHS))
def test_enumerate_parity(name):
    g = SUPPORT_GRAPHS[name]()
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    want = O.enumerate_triangles(g.n, crow, ccol).astype(np.int64)
    for v in VARIANTS:
        rp, cl = on_dev(g.rowptr, g.col)
        T, tri = tc.enumerate_triangles(rp, cl, force_variant=v)
        assert T == len(want), (name, v)
        assert (sorted_rows(np_u(tri, np.uint32)) == want).all(), (name, v)


def test_enumerate_capacity_host_and_prune():
    g = G.rmat(13, 16, seed=4)
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    want = O.enumerate_triangles(g.n, crow, ccol).astype(np.int64)
    T, tri = tc.enumerate_triangles(g.rowptr, g.col)               # host pointers
    assert T == len(want) and (sorted_rows(tri) == want).all()
    T0, _ = tc.enumerate_triangles(g.rowptr, g.col, capacity=0)    # count only
    assert T0 == len(want)
    k = len(want) // 3
    T1, part = tc.enumerate_triangles(g.rowptr, g.col, capacity=k)  # subset of size k
    assert T1 == len(want) and len(part) == k
    ws = {tuple(r) for r in want.tolist()}
    ps = {tuple(r) for r in part.astype(np.int64).tolist()}
    assert len(ps) == k and ps <= ws
    rp, cl = on_dev(crow, ccol)
    T2, tri2 = tc.enumerate_triangles(rp, cl, clean=True, sorted_rows=True, prune=True)
    assert T2 == len(want) and (sorted_rows(np_u(tri2, np.uint32)) == want).all()


def test_enumerate_rmat16_exact():
    g = G.rmat(16, 16)
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    want = O.enumerate_triangles(g.n, crow, ccol).astype(np.int64)
    rp, cl = on_dev(g.rowptr, g.col)
    T, tri = tc.enumerate_triangles(rp, cl)
    assert T == len(want) and (sorted_rows(np_u(tri, np.uint32)) == want).all()


def test_enumerate_rmat21_full_properties():
    """The bench workload: T triangles, all distinct, ascending, and sampled rows are triangles."""
    g = G.rmat(21, 16)
    T = O.count(g.n, g.rowptr, g.col)
    rp, cl = on_dev(g.rowptr, g.col)
    got, tri = tc.enumerate_triangles(rp, cl)
    assert got == T and tri.shape == (T, 3)
    t64 = tri.to(torch.int64)
    assert bool((t64[:, 0] < t64[:, 1]).all()) and bool((t64[:, 1] < t64[:, 2]).all())
    key = (t64[:, 0] << 42) | (t64[:, 1] << 21) | t64[:, 2]
    del t64
    key, _ = torch.sort(key)
    assert not bool((key[1:] == key[:-1]).any())                 # no triangle listed twice
    del key
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    rng = np.random.default_rng(2)
    rows = np_u(tri[torch.from_numpy(rng.integers(0, T, 2000)).to(DEV)], np.uint32)
    for a, b, c in rows.astype(np.int64):
        for x, y in ((a, b), (a, c), (b, c)):
            nx = ccol[crow[x]:crow[x + 1]]
            i = np.searchsorted(nx, y)
            assert i < len(nx) and nx[i] == y, (a, b, c)


# ------------------------------------------------------------------ NEXT-4: masked SpGEMM
@pytest.mark.parametrize("name", list(SUPPORT_GRAPHS))
@pytest.mark.parametrize("id_order", [False, True])
def test_masked_spgemm_parity(name, id_order):
    g = SUPPORT_GRAPHS[name]()
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    want_off, want_col, want_c, want_T = O.masked_spgemm(g.n, crow, ccol, id_order=id_order)
    for v in VARIANTS:
        rp, cl = on_dev(g.rowptr, g.col)
        off, colp, c, T = tc.masked_spgemm(rp, cl, id_order=id_order, force_variant=v)
        assert T == want_T, (name, id_order, v)
        assert (np_u(off, np.uint64) == want_off).all() and (np_u(colp, np.uint32) == want_col).all()
        assert (np_u(c, np.uint32) == want_c).all(), (name, id_order, v)


def test_masked_spgemm_fig_mm_printed(golden):
    """The GPU reproduces the paper's printed C in the figure's id order."""
    fx = golden("fig_mm.txt")
    C = np.array(fx["C"], dtype=np.int64)
    g = G.fig_mm()
    off, colp, c, T = tc.masked_spgemm(g.rowptr, g.col, id_order=True)   # host pointers
    assert T == 3
    got = np.zeros((7, 7), dtype=np.int64)
    src = np.repeat(np.arange(7), np.diff(off.astype(np.int64)))
    got[src, colp.astype(np.int64)] = c
    assert (got + got.T == C).all()


def test_id_order_counts_and_orientation():
    g = G.rmat(13, 16, seed=9)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    want_off, want_col = O.orient_order(g.n, crow, ccol, id_order=True)
    for clean in (False, True):
        rp, cl = on_dev(crow, ccol) if clean else on_dev(g.rowptr, g.col)
        off, colp = tc.orient(rp, cl, clean=clean, sorted_rows=clean, id_order=True)
        assert (np_u(off, np.uint64) == want_off).all() and (np_u(colp, np.uint32) == want_col).all()
        for v in VARIANTS:
            got, pv = tc.count_ex(rp, cl, clean=clean, sorted_rows=clean, id_order=True,
                                  per_vertex=True, force_variant=v)
            assert got == T and (np_u(pv, np.uint64) == t).all(), (clean, v)


def test_masked_spgemm_prune_host_and_rmat16():
    g = G.rmat(16, 16, seed=2)
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    for id_order in (False, True):
        want = O.masked_spgemm(g.n, crow, ccol, id_order=id_order)
        off, colp, c, T = tc.masked_spgemm(g.rowptr, g.col, id_order=id_order)
        assert T == want[3] and (off == want[0]).all() and (colp == want[1]).all() and (c == want[2]).all()
    prow, pcol, _ = O.prune(g.n, crow, ccol, 0)
    want = O.masked_spgemm(g.n, prow, pcol, id_order=False)
    rp, cl = on_dev(crow, ccol)
    off, colp, c, T = tc.masked_spgemm(rp, cl, clean=True, sorted_rows=True, prune=True)
    assert T == want[3] and (np_u(colp, np.uint32) == want[1]).all() and (np_u(c, np.uint32) == want[2]).all()
