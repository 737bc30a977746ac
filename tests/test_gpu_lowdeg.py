"""GPU parity of the bounded-degree path (csrc/lowdeg.cu, tc_options.lowdeg_max): graphs on
which every vertex has at most 32 arc incidences (road networks, meshes: P:700-702) are
cleaned, oriented and intersected by one thread per vertex.  Bit-exact T and t(v) against the
oracle on dirty and clean (sorted / unsorted) input, the eligibility boundary (exactly L
incidences vs L + 1, which must fall back to the general pipeline), the stats, the false
TC_CLEAN claim, and the full road mesh (BASELINE configs[3]).
"""
import numpy as np
import pytest

import graphgen as G
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1804_06926_b200 as tc  # noqa: E402

DEV = torch.device("cuda:0")
LD_MAX_LAUNCHES = 8        # the path launches <= 6 kernels (+ the scan); the pipeline ~40


def on_dev(rowptr, col):
    return (torch.from_numpy(np.ascontiguousarray(rowptr, np.uint64).view(np.int64)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(col, np.uint32).view(np.int32)).to(DEV))


def run(g_or_csr, **kw):
    rp, cl = (g_or_csr.rowptr, g_or_csr.col) if hasattr(g_or_csr, "rowptr") else g_or_csr
    out = tc.count_ex(*on_dev(rp, cl), per_vertex=True, with_stats=True, **kw)
    torch.cuda.synchronize()
    T, pv, st = out
    return T, pv.cpu().numpy().view(np.uint64), st


def clean_csr(g, sort=True, seed=0):
    """The simple symmetric CSR of g (the oracle's cleaning), rows ascending or shuffled."""
    row, col = O.clean(g.n, g.rowptr, g.col)
    if not sort:
        rng = np.random.default_rng(seed)
        col = col.copy()
        for u in range(g.n):
            rng.shuffle(col[row[u]:row[u + 1]])
    return row, col


def check(g, expect_lowdeg=True, **kw):
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    got, pv, st = run(g, **kw)
    assert got == T
    assert (pv[:g.n] == t).all()
    if expect_lowdeg is None:     # either path (duplicated arcs may push a hub over 32)
        pass
    elif expect_lowdeg:
        assert st["kernel_launches"] <= LD_MAX_LAUNCHES, st["kernel_launches"]
    else:
        assert st["kernel_launches"] > LD_MAX_LAUNCHES, st["kernel_launches"]
    return T, st


GRAPHS = {
    "mesh": lambda: G.road_mesh(200, 150, seed=3),
    "tri_grid": lambda: G.triangulated_grid(90, 70),
    "gnp_sparse": lambda: G.gnp(5000, 0.0012, seed=5),
    "cycle": lambda: G.cycle(3000),
    "tree": lambda: G.random_tree(4000, seed=2),
    "karate": lambda: G.karate(),
    "friendship": lambda: G.friendship(15),   # hub of degree 30 <= 32
    "union": lambda: G.disjoint_union(G.complete(12), G.cycle(500), G.road_mesh(60, 60, seed=1)),
}


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_lowdeg_dirty_parity(name):
    g = GRAPHS[name]()
    check(g, tiny_max_n=0)
    check(G.dirty(g, seed=7, dup=0.5, loops=20), tiny_max_n=0,
          expect_lowdeg=None if name in ("friendship", "karate") else True)


@pytest.mark.parametrize("name", sorted(GRAPHS))
@pytest.mark.parametrize("sort", [True, False])
def test_lowdeg_clean_parity(name, sort):
    g = GRAPHS[name]()
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    row, col = clean_csr(g, sort=sort, seed=3)
    got, pv, st = run((row, col), clean=True, sorted_rows=sort, tiny_max_n=0)
    assert got == T and (pv[:g.n] == t).all()
    assert st["kernel_launches"] <= LD_MAX_LAUNCHES


def test_triangulated_grid_closed_form():
    W, H = 301, 207
    g = G.triangulated_grid(W, H)
    got, _, _ = run(g)
    assert got == 2 * (W - 1) * (H - 1)


def _star_plus(k):
    """A star with k leaves plus a triangle on three leaves: the hub has k incidences."""
    e = [(0, i) for i in range(1, k + 1)] + [(1, 2), (2, 3), (1, 3)]
    return G.from_edges(k + 1 + 1500, e)   # isolated vertices: n > the one-kernel limit


@pytest.mark.parametrize("k,lowdeg", [(17, True), (31, True), (32, True), (33, False), (200, False)])
def test_eligibility_boundary(k, lowdeg):
    """Exactly 32 incidences stays on the path; 33 (as in-arcs or out-arcs) falls back."""
    g = _star_plus(k)
    check(g, expect_lowdeg=lowdeg)
    # the same star with every arc reversed (the hub's incidences are then in-arcs)
    s, d = g.arc_list()
    check(G.from_arcs(g.n, d, s), expect_lowdeg=lowdeg)
    # duplicated arcs count as incidences: 17 double arcs = 34 > 32 falls back, exact either way
    if k == 17:
        check(G.symmetric_arcs(g), expect_lowdeg=False)


def test_lowdeg_max_option():
    g = G.road_mesh(120, 120, seed=4)    # up to 8 incidences per vertex
    check(g, lowdeg_max=8)
    check(g, lowdeg_max=2, expect_lowdeg=False)
    check(g, lowdeg_max=0, expect_lowdeg=False)
    check(g, force_variant=tc.VARIANT_MERGE, expect_lowdeg=False)   # forced variants: pipeline


def test_lowdeg_stats_match_oracle_and_pipeline():
    g = G.dirty(G.road_mesh(300, 200, seed=8), seed=1)
    T, st_o = O.count(g.n, g.rowptr, g.col, with_stats=True)
    got, _, st = run(g)
    _, _, sp = run(g, lowdeg_max=0)                      # the general pipeline
    assert got == T
    assert st["m_undirected"] == st_o["m"] and st["work_W"] == st_o["W"]
    assert st["max_dplus"] == st_o["max_dplus"]
    assert st["work_stage"] == st_o["sum_dminus_dplus"]
    assert st["bytes_alg"] == 4 * st_o["W"] + 16 * st_o["m"]
    assert sum(st["bin_edges"]) + st["skipped_edges"] == st_o["m"]
    assert st["work_probe"] == sp["work_probe"] and st["skipped_edges"] == sp["skipped_edges"]


def test_lowdeg_host_pointers():
    g = G.dirty(G.road_mesh(150, 150, seed=2), seed=4)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    got, pv, st = tc.count_ex(g.rowptr, g.col, per_vertex=True, with_stats=True)
    assert got == T and (pv[:g.n] == t).all()
    assert st["kernel_launches"] <= LD_MAX_LAUNCHES


def test_lowdeg_false_clean_claim():
    """A one-way cycle claimed TC_CLEAN: n-1 arcs pass the rank filter > m/2 -> TC_EGRAPH."""
    n = 5000
    rp = np.arange(n + 1, dtype=np.uint64)
    cl = ((np.arange(n) + 1) % n).astype(np.uint32)
    with pytest.raises(tc.TCError) as e:
        run((rp, cl), clean=True)
    assert e.value.status == 2
    g = G.road_mesh(50, 50, seed=1)
    check(g)                              # the device is still sane


def test_lowdeg_empty_rows_and_isolated():
    n = 4096
    rp = np.zeros(n + 1, dtype=np.uint64)
    rp[2001:] = 3
    cl = np.array([5, 9, 7], dtype=np.uint32)    # vertex 2000: arcs to 5, 9, 7; no triangle
    got, pv, _ = run((rp, cl))
    assert got == 0 and not pv.any()
    g = G.from_edges(n, [(10, 11), (11, 12), (12, 10), (10, 10), (11, 10)])
    T, pv, st = run(g)
    assert T == 1 and pv[10] == pv[11] == pv[12] == 1 and st["m_undirected"] == 3


def test_config_road_full_both_paths():
    """BASELINE configs[3] (14 M vertices, 17 M edges): the bounded-degree path and the
    general pipeline both equal the oracle, per vertex."""
    g = G.road_mesh()
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    for kw in ({}, {"lowdeg_max": 0}):
        got, pv, st = run(g, **kw)
        assert got == T and (pv[:g.n] == t).all()
    row, col = clean_csr(g)
    got, pv, st = run((row, col), clean=True, sorted_rows=True)
    assert got == T and (pv[:g.n] == t).all() and st["kernel_launches"] <= LD_MAX_LAUNCHES
