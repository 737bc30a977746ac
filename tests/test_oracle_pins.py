"""Pins for the CPU oracle (oracle/) against things other than itself.

Every check here is fixed by the paper or by mathematics, never by the oracle:
  * the paper's worked example (Fig. mm): T = 3;
  * closed forms (K_n = C(n,3), wheels, trees / bipartite = 0, K_{a,b,c} = abc,
    friendship and windmill graphs, triangulated grids 2(W-1)(H-1));
  * Kronecker products: trace((B(x)C)^3) = trace(B^3) trace(C^3), hence
    T(B(x)C) = 6 T(B) T(C) and t(u1,u2) = 2 t_B(u1) t_C(u2);
  * brute force over all vertex triples (the definition) on tiny graphs;
  * trace(A^3)/6 and diag(A^3)/2 (a different mathematical route) on small graphs;
  * invariants: sum_v t(v) = 3T, 3T <= wedges, invariance under duplicates,
    self-loops, reversed arcs and relabelling; orientation invariants.
A plausible bug (dropped match, wrong tie rule, transposed operand, missing
symmetrisation, off-by-one in a row bound) fails at least one of these.
"""
import itertools
import math

import numpy as np
import pytest

import graphgen as G
import oracle as O


def dense(g):
    A = np.zeros((g.n, g.n), dtype=np.int64)
    s, d = g.arc_list()
    A[s, d] = 1
    A[d, s] = 1
    np.fill_diagonal(A, 0)
    return A


def brute_force(A):
    """Definition: count triples a<b<c with all three edges (O(n^3))."""
    n = A.shape[0]
    T = 0
    t = np.zeros(n, dtype=np.int64)
    for a, b, c in itertools.combinations(range(n), 3):
        if A[a, b] and A[b, c] and A[a, c]:
            T += 1
            t[a] += 1
            t[b] += 1
            t[c] += 1
    return T, t


def brute_force_fast(A):
    """Same definition vectorised over c: for a<b adjacent, count c>b adjacent to both."""
    n = A.shape[0]
    T = 0
    t = np.zeros(n, dtype=np.int64)
    for a in range(n):
        for b in range(a + 1, n):
            if A[a, b]:
                cs = np.nonzero(A[a, b + 1:] & A[b, b + 1:])[0] + b + 1
                T += cs.size
                t[a] += cs.size
                t[b] += cs.size
                t[cs] += 1
    return T, t


def trace_pin(A):
    A3 = A @ A @ A
    return int(np.trace(A3)) // 6, np.diag(A3) // 2


def oracle_T(g, pv=False):
    return O.count(g.n, g.rowptr, g.col, per_vertex=pv)


# ------------------------------------------------------------ the paper's example
def test_fig_mm_paper_example(golden):
    fx = golden("fig_mm.txt")
    A = np.array(fx["A"], dtype=np.int64)
    assert (A == A.T).all() and A.shape == (7, 7)
    g = G.from_edges(7, [(i, j) for i in range(7) for j in range(7) if A[i, j]])
    T, t = oracle_T(g, pv=True)
    assert T == fx["T"][0][0] == 3
    tris = fx["TRI"]
    for a, b, c in tris:                                   # the listed triples are triangles of A
        assert A[a, b] and A[b, c] and A[a, c]
    expect = np.zeros(7, dtype=np.int64)
    for tri in tris:
        expect[tri] += 1
    assert list(t) == list(expect)


def test_fig_mm_stats():
    T, st = O.count(7, *_csr(G.fig_mm()), with_stats=True)
    assert st["m"] == 10                                   # 20 directed edges (Table 1 convention)
    assert st["SSD"] == 62                                 # degrees [3,3,3,3,3,4,1]
    assert st["wedges"] == 21
    # SURVEY §8(c) worked example under rank orientation: N+ = {0:[1,4,5], 1:[2,5], 2:[3],
    # 3:[4,5], 4:[5], 5:[], 6:[2]} -> W = sum over oriented edges of d+u + d+v = 28
    assert st["W"] == 28
    assert st["max_dplus"] == 3 and st["max_deg"] == 4
    # d- = [0,1,2,1,2,4,0], d+ = [3,2,1,2,1,0,1] (d = d+ + d- = the degrees above):
    # sum d- d+ = 0+2+2+2+2+0+0 = 8
    assert st["sum_dminus_dplus"] == 8


def test_closed_form_stats():
    """Work statistics with closed forms (karate W = 302, max d+ 5; K_n:
    every oriented edge (i, j), i < j in rank order, has d+ = n-1-i and n-1-j)."""
    _, st = O.count(34, *_csr(G.karate()), with_stats=True)
    assert (st["m"], st["W"], st["SSD"], st["max_dplus"], st["max_deg"], st["wedges"]) == \
        (78, 302, 1212, 5, 17, 528)
    for n in (5, 20, 57):
        _, st = O.count(n, *_csr(G.complete(n)), with_stats=True)
        W = sum((n - 1 - i) + (n - 1 - j) for i in range(n) for j in range(i + 1, n))
        assert st["W"] == W and st["max_dplus"] == n - 1
        assert st["sum_dminus_dplus"] == sum(i * (n - 1 - i) for i in range(n))
    _, st = O.count(9, *_csr(G.star(8)), with_stats=True)   # leaves -> hub: d+ = 1, hub d+ = 0
    assert (st["W"], st["max_dplus"], st["sum_dminus_dplus"]) == (8, 1, 0)


@pytest.mark.parametrize("seed", [1, 2])
def test_work_stats_numpy(seed):
    """W, sum d- d+ and max d+ recomputed with numpy from the definition (rank = (d, id),
    orientation low -> high rank), independent of the oracle's C code."""
    g = G.gnp(300, 0.07, seed)
    src, dst = g.arc_list()
    keep = src != dst
    a = np.minimum(src[keep], dst[keep]).astype(np.int64)
    b = np.maximum(src[keep], dst[keep]).astype(np.int64)
    pairs = np.unique(a * g.n + b)
    a, b = pairs // g.n, pairs % g.n
    d = np.bincount(a, minlength=g.n) + np.bincount(b, minlength=g.n)
    a_low = (d[a] < d[b]) | ((d[a] == d[b]) & (a < b))
    u = np.where(a_low, a, b)
    v = np.where(a_low, b, a)
    dplus = np.bincount(u, minlength=g.n)
    dminus = np.bincount(v, minlength=g.n)
    _, st = O.count(g.n, g.rowptr, g.col, with_stats=True)
    assert st["m"] == len(pairs)
    assert st["W"] == int((dplus[u] + dplus[v]).sum())
    assert st["sum_dminus_dplus"] == int((dminus * dplus).sum())
    assert st["max_dplus"] == int(dplus.max())
    assert st["SSD"] == int((d * d).sum())


def _csr(g):
    return g.rowptr, g.col


def test_karate(golden):
    fx = golden("karate.txt")
    g = G.karate()
    T, t, st = O.count(g.n, g.rowptr, g.col, per_vertex=True, with_stats=True)
    assert T == fx["T"][0][0] == 45
    assert st["m"] == fx["M"][0][0]
    assert list(t) == fx["PV"][0]
    bf_T, bf_t = brute_force(dense(g))
    assert (bf_T, list(bf_t)) == (45, fx["PV"][0])
    assert int(t.sum()) == 3 * T


# ------------------------------------------------------------ closed forms
@pytest.mark.parametrize("n", list(range(1, 41)) + [100, 333])
def test_complete_graph(n):
    T, t = oracle_T(G.complete(n), pv=True)
    assert T == math.comb(n, 3)
    assert all(int(x) == math.comb(n - 1, 2) for x in t)


def test_complete_1000():
    assert oracle_T(G.complete(1000)) == 166_167_000


@pytest.mark.parametrize("n", range(5, 40))
def test_wheel(n):
    T, t = oracle_T(G.wheel(n), pv=True)
    assert T == n - 1                                      # n vertices, n >= 5 (DESIGN reading R10)
    assert int(t[0]) == n - 1 and all(int(x) == 2 for x in t[1:])


def test_wheel4_is_k4():
    assert oracle_T(G.wheel(4)) == 4


@pytest.mark.parametrize("n", range(3, 30))
def test_cycles_paths_stars(n):
    assert oracle_T(G.cycle(n)) == (1 if n == 3 else 0)
    assert oracle_T(G.path(n)) == 0
    assert oracle_T(G.star(n)) == 0


@pytest.mark.parametrize("seed", range(20))
def test_trees_and_bipartite_zero(seed):
    assert oracle_T(G.random_tree(50 + 13 * seed, seed)) == 0
    assert oracle_T(G.random_bipartite(10 + seed, 20, 0.4, seed)) == 0


@pytest.mark.parametrize("a,b,c", [(1, 1, 1), (2, 3, 4), (5, 5, 5), (1, 7, 9), (10, 20, 30)])
def test_complete_tripartite(a, b, c):
    assert oracle_T(G.complete_multipartite([a, b, c])) == a * b * c


def test_complete_bipartite_k33():
    assert oracle_T(G.complete_multipartite([3, 3])) == 0


@pytest.mark.parametrize("k", [1, 2, 5, 50])
def test_friendship_and_windmill(k):
    T, t = oracle_T(G.friendship(k), pv=True)
    assert T == k and int(t[0]) == k
    assert oracle_T(G.windmill(k, 6)) == k * math.comb(6, 3)


@pytest.mark.parametrize("W,H", [(2, 2), (5, 5), (37, 23), (300, 300)])
def test_triangulated_grid(W, H):
    assert oracle_T(G.triangulated_grid(W, H, seed=W)) == 2 * (W - 1) * (H - 1)


def test_disjoint_union_additive():
    parts = [G.complete(7), G.wheel(9), G.karate(), G.fig_mm()]
    assert oracle_T(G.disjoint_union(*parts)) == sum(oracle_T(p) for p in parts)


# ------------------------------------------------------------ Kronecker products
def test_kronecker_products():
    pairs = [(G.karate(), G.karate()), (G.karate(), G.complete(5)), (G.fig_mm(), G.karate()),
             (G.wheel(6), G.fig_mm())]
    for B, C in pairs:
        TB, tB = oracle_T(B, pv=True)
        TC, tC = oracle_T(C, pv=True)
        A = G.kron(B, C)
        TA, tA = oracle_T(A, pv=True)
        assert TA == 6 * TB * TC
        assert (tA == 2 * np.outer(tB, tC).reshape(-1)).all()


def test_karate_cubed():
    g = G.kron_power(G.karate(), 3)
    T, st = O.count(g.n, g.rowptr, g.col, with_stats=True)
    assert g.n == 39304
    assert st["m"] == 2 ** 2 * 78 ** 3 == 1_898_208         # m = 2^(k-1) 78^k
    assert T == 6 ** 2 * 45 ** 3 == 3_280_500


# ------------------------------------------------------------ brute force / trace
@pytest.mark.parametrize("seed", range(60))
def test_brute_force_gnp(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(4, 45))
    p = [0.02, 0.1, 0.3, 0.6][seed % 4]
    g = G.gnp(n, p, seed)
    T, t = oracle_T(g, pv=True)
    bT, bt = brute_force(dense(g))
    assert T == bT and list(t) == list(bt)


@pytest.mark.parametrize("seed", range(40))
def test_trace_gnp(seed):
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(50, 400))
    p = [0.02, 0.05, 0.1, 0.3][seed % 4]
    g = G.gnp(n, p, seed)
    T, t = oracle_T(g, pv=True)
    tT, tt = trace_pin(dense(g))
    assert T == tT and (t == tt).all()


@pytest.mark.parametrize("scale", [6, 8, 9])
def test_trace_rmat(scale):
    g = G.rmat(scale, 16, seed=scale)                     # raw arcs: dups, loops, one direction
    T, t = oracle_T(g, pv=True)
    tT, tt = trace_pin(dense(g))
    assert T == tT and (t == tt).all()
    if scale <= 8:
        bT, bt = brute_force_fast(dense(g))
        assert T == bT and (t == bt).all()


def test_trace_chung_lu_small():
    g = G.chung_lu(n=700, npairs=6000, seed=3)
    T, t = oracle_T(g, pv=True)
    tT, tt = trace_pin(dense(g))
    assert T == tT and (t == tt).all() and T > 0


def test_trace_clique_union_small():
    g = G.clique_union(n=500, groups=120, seed=9)
    T, t = oracle_T(g, pv=True)
    tT, tt = trace_pin(dense(g))
    assert T == tT and (t == tt).all() and T > 0


def test_trace_road_small():
    g = G.road_mesh(30, 25, 0.56, 0.3, seed=4)
    T, t = oracle_T(g, pv=True)
    tT, tt = trace_pin(dense(g))
    assert T == tT and (t == tt).all()


# ------------------------------------------------------------ invariants
@pytest.mark.parametrize("seed", range(10))
def test_dirty_and_relabel_invariance(seed):
    g = G.rmat(9, 8, seed=100 + seed)
    T, t = oracle_T(g, pv=True)
    assert oracle_T(G.dirty(g, seed)) == T
    assert oracle_T(G.symmetric_arcs(g)) == T
    rng = np.random.default_rng(seed)
    perm = rng.permutation(g.n)
    s, d = g.arc_list()
    h = G.from_arcs(g.n, perm[s], perm[d])
    Th, th = oracle_T(h, pv=True)
    assert Th == T and (th[perm] == t).all()
    assert int(t.sum()) == 3 * T


def test_wedge_bound_and_ssd():
    for g in [G.karate(), G.rmat(10, 16), G.complete(30), G.gnp(200, 0.1, 1)]:
        T, st = O.count(g.n, g.rowptr, g.col, with_stats=True)
        A = dense(g)
        d = A.sum(1)
        assert st["wedges"] == int((d * (d - 1) // 2).sum())
        assert st["SSD"] == int((d * d).sum())
        assert 3 * T <= st["wedges"]
        assert st["m"] == int(A.sum()) // 2


def test_clean_matches_edge_set():
    g = G.dirty(G.rmat(10, 16, seed=5), 5)
    row, col = O.clean(g.n, g.rowptr, g.col)
    A = dense(g)
    # symmetric, sorted, loop-free, and exactly the edge set of A
    src = np.repeat(np.arange(g.n), np.diff(row).astype(np.int64))
    assert (A[src, col] == 1).all() and int(row[-1]) == int(A.sum())
    for u in range(g.n):
        r = col[row[u]:row[u + 1]]
        assert (np.diff(r.astype(np.int64)) > 0).all() and u not in r


def test_orient_invariants():
    for g in [G.rmat(11, 16, seed=3), G.karate(), G.complete(50), G.chung_lu(2000, 20000, seed=1)]:
        row, col = O.clean(g.n, g.rowptr, g.col)
        off, cp = O.orient(g.n, row, col)
        deg = np.diff(row).astype(np.int64)
        m = int(row[-1]) // 2
        assert cp.size == m and int(off[-1]) == m            # |E+| = m
        src = np.repeat(np.arange(g.n), np.diff(off).astype(np.int64))
        rank_u = deg[src] * (g.n + 1) + src
        rank_v = deg[cp] * (g.n + 1) + cp.astype(np.int64)
        assert (rank_u < rank_v).all()                        # acyclic total order
        dplus = np.diff(off).astype(np.int64)
        assert dplus.max(initial=0) ** 2 <= 2 * m             # d+ <= sqrt(2m)
        for u in range(g.n):
            r = cp[off[u]:off[u + 1]].astype(np.int64)
            assert (np.diff(r) > 0).all()
        # every undirected edge appears exactly once
        a = np.minimum(src, cp)
        b = np.maximum(src, cp)
        assert np.unique(a * g.n + b).size == m


def test_forward_is_order_independent():
    """Forward counts each triangle once under ANY total order."""
    for g in [G.rmat(10, 16, seed=8), G.karate(), G.complete(25)]:
        T = oracle_T(g)
        row, col = O.clean(g.n, g.rowptr, g.col)
        src = np.repeat(np.arange(g.n), np.diff(row).astype(np.int64))
        keep = src < col                                      # orient by id only
        off = np.zeros(g.n + 1, dtype=np.uint64)
        np.add.at(off, src[keep] + 1, 1)
        off = np.cumsum(off).astype(np.uint64)
        assert O.forward(g.n, off, col[keep]) == T


def test_vertex_triangles_definition(golden):
    g = G.karate()
    row, col = O.clean(g.n, g.rowptr, g.col)
    assert [O.vertex_triangles(g.n, row, col, v) for v in range(34)] == golden("karate.txt")["PV"][0]
    h = G.rmat(11, 16, seed=2)
    T, t = oracle_T(h, pv=True)
    row, col = O.clean(h.n, h.rowptr, h.col)
    for v in range(0, h.n, 37):
        assert O.vertex_triangles(h.n, row, col, v) == int(t[v])


def test_empty_and_degenerate():
    assert O.count(0, np.zeros(1, np.uint64), np.zeros(0, np.uint32)) == 0
    assert O.count(5, np.zeros(6, np.uint64), np.zeros(0, np.uint32)) == 0
    g = G.from_edges(3, [(0, 0), (1, 1), (0, 1), (1, 0), (0, 1)])
    assert oracle_T(g) == 0
    g = G.from_edges(3, [(0, 1), (1, 2), (2, 0), (2, 2), (0, 1)])
    assert oracle_T(g) == 1


def test_bad_input_rejected():
    with pytest.raises(ValueError):
        O.count(2, np.array([0, 1, 1], np.uint64), np.array([5], np.uint32))


# ------------------------------------------------------------------ NEXT-1: clustering
# Conventions (SURVEY §8(c) reading 9, R14): c(v) = 2t(v)/(d(v)(d(v)-1)),
# 0 for d(v) < 2; transitivity = 3T / sum_v C(d(v),2); average over all n vertices.
def test_clustering_karate_published():
    """Karate: transitivity 0.25568 and average clustering 0.57064 (SURVEY §8(c)
    reading 9, measured with networkx); T = 45 and 528 wedges give 135/528 exactly."""
    g = G.karate()
    cc, s = O.clustering(g.n, g.rowptr, g.col)
    assert s["triangles"] == 45 and s["wedges"] == 528
    assert s["transitivity"] == 135 / 528
    assert round(s["transitivity"], 5) == 0.25568
    assert round(s["avg_clustering"], 5) == 0.57064
    assert cc[0] == 0.15          # vertex 0: d = 16, t = 18 -> 36 / 240
    assert cc[11] == 0.0          # vertex 11: d = 1 -> 0 by convention


@pytest.mark.parametrize("n", [3, 4, 7, 20])
def test_clustering_complete(n):
    g = G.complete(n)
    cc, s = O.clustering(g.n, g.rowptr, g.col)
    assert (cc == 1.0).all() and s["transitivity"] == 1.0 and s["avg_clustering"] == 1.0
    assert s["wedges"] == n * math.comb(n - 1, 2)


@pytest.mark.parametrize("n", [5, 6, 9, 30])
def test_clustering_wheel(n):
    """Wheel with n vertices (hub 0 + rim cycle of n-1, n >= 5): hub c = 2/(n-2),
    rim c = 2/3; transitivity 3(n-1) / (C(n-1,2) + 3(n-1))."""
    g = G.wheel(n)
    cc, s = O.clustering(g.n, g.rowptr, g.col)
    hub = int(np.argmax(np.diff(g_clean_rowptr(g))))
    assert cc[hub] == 2.0 / (n - 2)
    assert all(cc[v] == 2.0 / 3.0 for v in range(n) if v != hub)
    assert s["wedges"] == math.comb(n - 1, 2) + 3 * (n - 1)
    assert s["transitivity"] == 3.0 * (n - 1) / (math.comb(n - 1, 2) + 3 * (n - 1))


def g_clean_rowptr(g):
    return O.clean(g.n, g.rowptr, g.col)[0]


@pytest.mark.parametrize("k", [1, 2, 5, 12])
def test_clustering_friendship(k):
    """F_k: centre d = 2k, t = k -> 1/(2k-1); every other vertex d = 2, t = 1 -> 1."""
    g = G.friendship(k)
    cc, s = O.clustering(g.n, g.rowptr, g.col)
    deg = np.diff(g_clean_rowptr(g))
    centre = int(np.argmax(deg))
    assert cc[centre] == 1.0 / (2 * k - 1) if k > 1 else cc[centre] == 1.0
    assert all(cc[v] == 1.0 for v in range(g.n) if v != centre)


def test_clustering_multipartite_and_zero_cases():
    """K_{a,b,c}: a vertex of part A has d = b+c, t = bc; trees and stars are 0;
    isolated vertices count 0 in the average."""
    a, b, c = 2, 3, 4
    g = G.complete_multipartite([a, b, c])
    cc, s = O.clustering(g.n, g.rowptr, g.col)
    want = {a: 2 * b * c / ((b + c) * (b + c - 1)), b: 2 * a * c / ((a + c) * (a + c - 1)),
            c: 2 * a * b / ((a + b) * (a + b - 1))}
    sizes = [a] * a + [b] * b + [c] * c
    assert all(cc[v] == want[sizes[v]] for v in range(g.n))
    wedges = a * math.comb(b + c, 2) + b * math.comb(a + c, 2) + c * math.comb(a + b, 2)
    assert s["wedges"] == wedges and s["transitivity"] == 3 * a * b * c / wedges
    for h in (G.star(9), G.random_tree(50, seed=3), G.path(7)):
        cc, s = O.clustering(h.n, h.rowptr, h.col)
        assert (cc == 0).all() and s["transitivity"] == 0.0 and s["avg_clustering"] == 0.0
    k4 = G.complete(4)
    iso = G.from_edges(10, np.stack(k4.arc_list(), 1))     # K4 + 6 isolated vertices
    cc, s = O.clustering(iso.n, iso.rowptr, iso.col)
    assert s["avg_clustering"] == 4 / 10 and (cc[4:] == 0).all()


def test_clustering_matches_dense_definition():
    """A different route: d = row sums of A, t = diag(A^3)/2 on small random graphs."""
    for seed in range(4):
        g = G.gnp(60, 0.15, seed=seed)
        A = dense(g)
        d = A.sum(1)
        t = np.diag(A @ A @ A) // 2
        cc, s = O.clustering(g.n, g.rowptr, g.col)
        want = np.where(d >= 2, 2.0 * t / np.maximum(d * (d - 1), 1), 0.0)
        assert (cc == want).all()
        assert s["wedges"] == int((d * (d - 1) // 2).sum())
