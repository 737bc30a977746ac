"""Pins for the NEXT-2 / NEXT-3 oracle functions (oracle.prune, oracle.edge_support,
oracle.enumerate_triangles) against things other than the oracle itself:

  * closed forms: paths, cycles, stars, trees, lollipops (K_5 plus a pendant path)
    under k rounds of leaf pruning; support n-2 on K_n, 2 / 1 on wheel spokes / rims,
    1 on friendship and windmill edges of K_3 blades, s-2 on windmill K_s blades;
  * the paper's worked example (Fig. mm): its three triangles, and the
    supports they imply;
  * an independent algorithm: the 2-core by a degree-queue peel (one vertex at a
    time, not the paper's rounds), compared edge for edge at the fixed point;
  * a different mathematical route: sup(u,v) = (A^2)[u,v] for every edge (numpy
    matmul), sum of supports = 3T = trace(A^3)/2;
  * brute force over all vertex triples (itertools) for enumeration;
  * invariants: T and t(v) unchanged by pruning; each round only deletes edges;
    every edge of a triangle survives every round.
A plausible bug (pruning on the old degrees of a later round, an off-by-one in the
degree threshold, supports counted through one endpoint only, a triangle listed
twice or with unsorted ids) fails at least one of these.
"""
import collections
import itertools
import math

import numpy as np
import pytest

import graphgen as G
import oracle as O


def clean(g):
    return O.clean(g.n, g.rowptr, g.col)


def edge_set(n, rowptr, col):
    s = set()
    for u in range(n):
        for v in col[rowptr[u]:rowptr[u + 1]]:
            s.add((min(u, int(v)), max(u, int(v))))
    return s


def dense(g):
    A = np.zeros((g.n, g.n), dtype=np.int64)
    s, d = g.arc_list()
    A[s, d] = 1
    A[d, s] = 1
    np.fill_diagonal(A, 0)
    return A


def lollipop(L):
    """K_5 on 0..4 plus the path 4 - 5 - ... - (4 + L)."""
    e = [(i, j) for i in range(5) for j in range(i + 1, 5)]
    e += [(4 + i, 5 + i) for i in range(L)]
    return G.from_edges(5 + L, e, f"lollipop{L}")


def two_core_peel(n, edges):
    """Independent 2-core: repeatedly remove ONE vertex of degree < 2 (queue)."""
    adj = collections.defaultdict(set)
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    q = collections.deque(v for v in range(n) if len(adj[v]) < 2)
    gone = set()
    while q:
        v = q.popleft()
        if v in gone:
            continue
        gone.add(v)
        for w in list(adj[v]):
            adj[w].discard(v)
            if len(adj[w]) < 2 and w not in gone:
                q.append(w)
        adj[v].clear()
    return {(a, b) for a, b in edges if a not in gone and b not in gone}


# ------------------------------------------------------------------ NEXT-2: pruning
@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 17])
@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_prune_path_rounds(n, k):
    g = G.path(n)
    r, c, done = O.prune(n, *clean(g), rounds=k)
    assert done == k
    assert int(r[n]) // 2 == max(0, n - 1 - 2 * k)     # each round strips both end edges


@pytest.mark.parametrize("n", [2, 3, 6, 9, 20])
def test_prune_path_fixed_point(n):
    r, c, done = O.prune(n, *clean(G.path(n)), rounds=0)
    assert int(r[n]) == 0
    assert done == math.ceil((n - 1) / 2) + 1          # + the final round that deletes nothing


@pytest.mark.parametrize("n", [3, 4, 10])
def test_prune_cycle_untouched(n):
    crow, ccol = clean(G.cycle(n))
    r, c, done = O.prune(n, crow, ccol, rounds=0)
    assert done == 1 and (r == crow).all() and (c == ccol).all()


@pytest.mark.parametrize("L", [1, 2, 7])
def test_prune_lollipop(L):
    g = lollipop(L)
    for k in range(1, L + 1):
        r, c, _ = O.prune(g.n, *clean(g), rounds=k)
        assert int(r[g.n]) // 2 == 10 + L - k           # one pendant edge per round
    r, c, done = O.prune(g.n, *clean(g), rounds=0)
    assert edge_set(g.n, r, c) == {(i, j) for i in range(5) for j in range(i + 1, 5)}
    assert done == L + 1


@pytest.mark.parametrize("seed", range(4))
def test_prune_trees_and_stars_vanish(seed):
    t = G.random_tree(60 + seed, seed)
    r, _, _ = O.prune(t.n, *clean(t), rounds=0)
    assert int(r[t.n]) == 0
    s = G.star(9)
    r, _, done = O.prune(s.n, *clean(s), rounds=1)
    assert int(r[s.n]) == 0 and done == 1


@pytest.mark.parametrize("g", [G.gnp(80, 0.03, 1), G.gnp(120, 0.02, 2), G.rmat(9, 4),
                               G.road_mesh(40, 40, seed=3), G.random_tree(50, 5)],
                         ids=lambda g: g.name)
def test_prune_fixed_point_is_two_core(g):
    crow, ccol = clean(g)
    r, c, _ = O.prune(g.n, crow, ccol, rounds=0)
    assert edge_set(g.n, r, c) == two_core_peel(g.n, edge_set(g.n, crow, ccol))
    # rows stay sorted and symmetric
    for u in range(g.n):
        row = c[r[u]:r[u + 1]]
        assert (np.diff(row.astype(np.int64)) > 0).all()


@pytest.mark.parametrize("g", [G.gnp(90, 0.04, 7), G.rmat(10, 8), G.road_mesh(30, 30, seed=4),
                               G.karate()], ids=lambda g: g.name)
def test_prune_keeps_triangles(g):
    crow, ccol = clean(g)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    prev = edge_set(g.n, crow, ccol)
    A = dense(g)
    tri_edges = {(a, b) for a, b in prev if (A[a] & A[b]).any()}
    for k in (1, 2, 3, 0):
        r, c, _ = O.prune(g.n, crow, ccol, rounds=k)
        es = edge_set(g.n, r, c)
        assert tri_edges <= es                         # every triangle edge survives
        if k:
            assert es <= prev                          # rounds only delete
            prev = es
        T2, t2 = O.count(g.n, r, c, per_vertex=True)
        assert T2 == T and (t2 == t).all()


def test_prune_round_uses_current_degrees():
    # path 0-1-2-3 with a triangle 3-4-5: round 1 deletes (0,1) only, round 2 (1,2),
    # round 3 (2,3); a variant that reused round-1 degrees would stop after round 1
    g = G.from_edges(6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (3, 5)])
    sizes = [int(O.prune(6, *clean(g), rounds=k)[0][6]) // 2 for k in (1, 2, 3, 4)]
    assert sizes == [5, 4, 3, 3]


# ------------------------------------------------------------------ NEXT-3: support
def support_of(g):
    crow, ccol = clean(g)
    off, colp = O.orient(g.n, crow, ccol)
    sup = O.edge_support(g.n, crow, ccol, off, colp)
    return off, colp, sup


def support_map(n, off, colp, sup):
    out = {}
    for u in range(n):
        for e in range(int(off[u]), int(off[u + 1])):
            v = int(colp[e])
            out[(min(u, v), max(u, v))] = int(sup[e])
    return out


@pytest.mark.parametrize("n", [2, 3, 4, 7, 12])
def test_support_complete(n):
    off, colp, sup = support_of(G.complete(n))
    assert len(sup) == n * (n - 1) // 2 and (sup == n - 2).all()


@pytest.mark.parametrize("n", [5, 6, 9, 20])
def test_support_wheel(n):
    g = G.wheel(n)
    sm = support_map(n, *support_of(g))
    for (a, b), s in sm.items():
        assert s == (2 if a == 0 else 1)               # spokes in 2 triangles, rim in 1


@pytest.mark.parametrize("k,s", [(1, 3), (4, 3), (3, 5), (2, 6)])
def test_support_windmill(k, s):
    g = G.windmill(k, s)
    off, colp, sup = support_of(g)
    assert (sup == s - 2).all()


def test_support_fig_mm(golden):
    fx = golden("fig_mm.txt")
    g = G.fig_mm()
    want = collections.Counter()
    for a, b, c in fx["TRI"]:                          # the paper's three triangles
        for x, y in ((a, b), (a, c), (b, c)):
            want[(x, y)] += 1
    sm = support_map(7, *support_of(g))
    assert {e: s for e, s in sm.items() if s} == dict(want)
    assert sum(sm.values()) == 3 * fx["T"][0][0]


@pytest.mark.parametrize("g", [G.gnp(70, 0.1, 3), G.rmat(9, 8), G.karate(),
                               G.dirty(G.gnp(50, 0.2, 4), seed=2), G.clique_union(2000, 900, seed=1)],
                         ids=lambda g: g.name)
def test_support_is_A_squared(g):
    Af = dense(g).astype(np.float64)                   # exact: entries < 2^53
    A2 = Af @ Af
    off, colp, sup = support_of(g)
    src = np.repeat(np.arange(g.n), np.diff(off.astype(np.int64)))
    assert (sup.astype(np.int64) == A2[src, colp.astype(np.int64)].astype(np.int64)).all()
    assert int(sup.sum()) == int(round(np.trace(A2 @ Af))) // 2   # 3T = trace(A^3)/2


def test_support_trees_zero():
    off, colp, sup = support_of(G.random_tree(40, 1))
    assert len(sup) == 39 and not sup.any()


# ------------------------------------------------------------------ NEXT-3: enumeration
@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 9, 15])
def test_enumerate_complete(n):
    g = G.complete(n) if n else G.from_edges(0, [])
    tri = O.enumerate_triangles(g.n, *clean(g))
    assert [tuple(map(int, t)) for t in tri] == list(itertools.combinations(range(n), 3))


def test_enumerate_fig_mm(golden):
    fx = golden("fig_mm.txt")
    tri = O.enumerate_triangles(7, *clean(G.fig_mm()))
    assert [list(map(int, t)) for t in tri] == fx["TRI"]


@pytest.mark.parametrize("seed", range(4))
def test_enumerate_brute_force(seed):
    g = G.gnp(26, 0.3, 40 + seed)
    A = dense(g)
    want = [t for t in itertools.combinations(range(g.n), 3)
            if A[t[0], t[1]] and A[t[1], t[2]] and A[t[0], t[2]]]
    got = [tuple(map(int, t)) for t in O.enumerate_triangles(g.n, *clean(g))]
    assert got == want


@pytest.mark.parametrize("n", [5, 8, 30])
def test_enumerate_wheel_closed_form(n):
    tri = O.enumerate_triangles(n, *clean(G.wheel(n)))
    assert len(tri) == n - 1 and (tri[:, 0] == 0).all()
    assert (tri[:, 0] < tri[:, 1]).all() and (tri[:, 1] < tri[:, 2]).all()


# ------------------------------------------------------------------ NEXT-4: masked SpGEMM
def test_masked_spgemm_fig_mm(golden):
    """Alg. 3 on the paper's worked example reproduces the printed B and C."""
    fx = golden("fig_mm.txt")
    A = np.array(fx["A"], dtype=np.int64)
    B = np.array(fx["B"], dtype=np.int64)
    C = np.array(fx["C"], dtype=np.int64)
    L, U = np.tril(A, -1), np.triu(A, 1)
    assert (L @ U == B).all() and (A * B == C).all()      # the transcription is consistent
    assert C.sum() // 2 == fx["T"][0][0] == 3
    g = G.fig_mm()
    off, colp, c, T = O.masked_spgemm(7, *clean(g), id_order=True)
    assert T == 3
    for i in range(7):
        for e in range(int(off[i]), int(off[i + 1])):
            j = int(colp[e])
            assert j > i and c[e] == C[i, j]
    assert sum(int(x) for x in c) == C.sum() // 2            # upper triangle only


def perm_order(A, id_order):
    d = A.sum(1)
    return np.arange(len(d)) if id_order else np.lexsort((np.arange(len(d)), d))


@pytest.mark.parametrize("id_order", [True, False])
@pytest.mark.parametrize("g", [G.gnp(60, 0.15, 8), G.rmat(8, 8), G.karate(), G.wheel(12),
                               G.clique_union(500, 300, seed=3), G.road_mesh(12, 12, seed=1)],
                         ids=lambda g: g.name)
def test_masked_spgemm_dense_route(g, id_order):
    """C = A o (L U) by dense numpy matmul on the permuted matrix (Alg. 3 lines 1-4)."""
    A = np.zeros((g.n, g.n), dtype=np.int64)
    s, d = g.arc_list()
    A[s, d] = 1
    A[d, s] = 1
    np.fill_diagonal(A, 0)
    order = perm_order(A, id_order)                         # line 1: rows by nonzeros
    pos = np.empty(g.n, dtype=np.int64)
    pos[order] = np.arange(g.n)
    Ap = A[np.ix_(order, order)].astype(np.float64)
    Cp = Ap * (np.tril(Ap, -1) @ np.triu(Ap, 1))           # lines 2-4
    off, colp, c, T = O.masked_spgemm(g.n, *clean(g), id_order=id_order)
    src = np.repeat(np.arange(g.n), np.diff(off.astype(np.int64)))
    assert (pos[src] < pos[colp.astype(np.int64)]).all()    # upper triangle in that order
    assert (c.astype(np.int64) == Cp[pos[src], pos[colp.astype(np.int64)]].astype(np.int64)).all()
    assert T == int(round(Cp.sum())) // 2 == O.count(g.n, g.rowptr, g.col)
