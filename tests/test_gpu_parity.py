"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

All counts are integers: the bar is bit-exact equality of T, of every t(v),
and of the oriented CSR (off+, col+) produced by steps a1-a4.
"""
import math

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


def gpu_count(rowptr, col, **kw):
    rp, cl = on_dev(rowptr, col)
    out = tc.count_ex(rp, cl, **kw)
    torch.cuda.synchronize()
    return out


def pv_np(t):
    return t.cpu().numpy().view(np.uint64)


def check_graph(g, variants=VARIANTS, per_vertex=True, **kw):
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    for v in variants:
        if per_vertex:
            got, pv = gpu_count(g.rowptr, g.col, per_vertex=True, force_variant=v, **kw)
            assert got == T, (g.name, v, got, T)
            assert (pv_np(pv) == t).all(), (g.name, v)
        else:
            assert gpu_count(g.rowptr, g.col, force_variant=v, **kw) == T, (g.name, v)
    return T


# ------------------------------------------------------------------ fixtures / closed forms
def test_fixtures(golden):
    assert check_graph(G.fig_mm()) == golden("fig_mm.txt")["T"][0][0] == 3
    assert check_graph(G.karate()) == golden("karate.txt")["T"][0][0] == 45
    assert check_graph(G.complete(20)) == 1140
    assert check_graph(G.wheel(10)) == 9


def test_degenerate():
    assert gpu_count(np.zeros(1, np.uint64), np.zeros(0, np.uint32)) == 0            # n = 0
    T, pv = gpu_count(np.zeros(6, np.uint64), np.zeros(0, np.uint32), per_vertex=True)
    assert T == 0 and (pv_np(pv) == 0).all()                                         # m = 0
    for g in [G.from_edges(2, [(0, 1)]), G.from_edges(3, [(0, 1), (1, 2), (2, 0)]),
              G.from_edges(4, [(0, 0), (1, 1), (2, 2)]), G.path(50), G.star(300),
              G.from_edges(10, [(3, 4), (4, 5), (5, 3), (3, 4), (4, 3)])]:
        check_graph(g)


@pytest.mark.parametrize("n", [3, 4, 5, 33, 64, 65, 200, 700])
def test_complete(n):
    assert check_graph(G.complete(n), per_vertex=n <= 200) == math.comb(n, 3)


def test_closed_forms_mix():
    assert check_graph(G.complete_multipartite([5, 6, 7])) == 210
    assert check_graph(G.friendship(40)) == 40
    assert check_graph(G.windmill(30, 8)) == 30 * 56
    assert check_graph(G.random_bipartite(60, 70, 0.3, 1)) == 0
    assert check_graph(G.random_tree(5000, 3)) == 0
    assert check_graph(G.triangulated_grid(123, 77)) == 2 * 122 * 76


# ------------------------------------------------------------------ random graphs
@pytest.mark.parametrize("seed", range(24))
def test_gnp_dirty(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(4, 600))
    p = [0.005, 0.02, 0.1, 0.3][seed % 4]
    check_graph(G.dirty(G.gnp(n, p, seed), seed))


@pytest.mark.parametrize("scale", [8, 10, 12, 14])
def test_rmat_all_variants(scale):
    check_graph(G.rmat(scale, 16, seed=scale))


@pytest.mark.parametrize("kw", [dict(short_max=1), dict(short_max=1 << 31), dict(skew_ratio=1),
                                dict(skew_ratio=1 << 31), dict(hub_min_dplus=2),
                                dict(hub_min_dplus=1 << 31), dict(short_max=4, skew_ratio=2, hub_min_dplus=8)])
def test_threshold_invariance(kw):
    """The count is invariant under any bin thresholds."""
    check_graph(G.rmat(13, 16, seed=77), variants=[None], **kw)


def test_generators_small():
    check_graph(G.chung_lu(20000, 150000, seed=3))
    check_graph(G.clique_union(5000, 4000, seed=4))
    check_graph(G.road_mesh(200, 150, seed=5))
    check_graph(G.kron(G.karate(), G.karate()))


# ------------------------------------------------------------------ clean-input paths, orientation
def clean_csr(g):
    return O.clean(g.n, g.rowptr, g.col)


def shuffled_rows(n, row, col, seed):
    rng = np.random.default_rng(seed)
    col = col.copy()
    for u in range(n):
        a, b = int(row[u]), int(row[u + 1])
        col[a:b] = rng.permutation(col[a:b])
    return col


@pytest.mark.parametrize("name", ["rmat12", "karate", "K300", "gnp"])
def test_orientation_parity(name):
    g = {"rmat12": lambda: G.rmat(12, 16, seed=3), "karate": G.karate,
         "K300": lambda: G.complete(300), "gnp": lambda: G.gnp(500, 0.05, 2)}[name]()
    row, col = clean_csr(g)
    want_off, want_col = O.orient(g.n, row, col)
    cases = [dict(rowptr=g.rowptr, col=g.col),                                   # a1 path
             dict(rowptr=row, col=col, clean=True, sorted_rows=True),             # sorted clean
             dict(rowptr=row, col=shuffled_rows(g.n, row, col, 1), clean=True),   # a4 row sort
             dict(rowptr=row, col=shuffled_rows(g.n, row, col, 2), clean=True, allocator="library")]
    for c in cases:
        rp, cl = on_dev(c.pop("rowptr"), c.pop("col"))
        off, colp = tc.orient(rp, cl, **c)
        torch.cuda.synchronize()
        assert (off.cpu().numpy().view(np.uint64) == want_off).all(), (name, c)
        assert (colp.cpu().numpy().view(np.uint32) == want_col).all(), (name, c)


@pytest.mark.parametrize("scale", [10, 13])
def test_clean_input_counts(scale):
    g = G.rmat(scale, 16, seed=scale + 5)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    row, col = clean_csr(g)
    for kw in [dict(clean=True, sorted_rows=True), dict(clean=True),
               dict(clean=True, allocator="library")]:
        c = shuffled_rows(g.n, row, col, scale) if not kw.get("sorted_rows") else col
        for v in VARIANTS:
            got, pv = gpu_count(row, c, per_vertex=True, force_variant=v, **kw)
            assert got == T and (pv_np(pv) == t).all(), (kw, v)


def test_host_pointer_path():
    g = G.rmat(12, 16, seed=9)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    got, pv, st = tc.count_ex(g.rowptr, g.col, per_vertex=True, with_stats=True)
    assert got == T and (pv == t).all()
    assert st["h2d_bytes"] == g.rowptr.nbytes + g.col.nbytes
    assert st["d2h_bytes"] == 8 + 8 * g.n


def test_stats_consistent():
    g = G.rmat(12, 16, seed=4)
    T, st_o = O.count(g.n, g.rowptr, g.col, with_stats=True)
    got, st = gpu_count(g.rowptr, g.col, with_stats=True)
    assert got == T
    assert st["m_undirected"] == st_o["m"] and st["work_W"] == st_o["W"]
    assert st["max_dplus"] == st_o["max_dplus"]
    assert st["bytes_alg"] == 4 * st_o["W"] + 16 * st_o["m"]
    # the bins, the dense-core edges and the skipped edges partition the edge set
    assert sum(st["bin_edges"]) + st["core_edges"] + st["skipped_edges"] == st_o["m"]
    assert st["work_stage"] == st_o["sum_dminus_dplus"]          # SURVEY 8(d) B_stage
    assert st["kernel_launches"] > 0


# ------------------------------------------------------------------ multi-GPU partition (on one GPU)
@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_sum_to_total(world):
    g = G.rmat(12, 16, seed=21)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    rp, cl = on_dev(g.rowptr, g.col)
    tot, pv_sum, parts = 0, torch.zeros(g.n, dtype=torch.int64, device=DEV), []
    for r in range(world):
        partial = torch.zeros(1, dtype=torch.int64, device=DEV)
        pv = torch.zeros(g.n, dtype=torch.int64, device=DEV)
        tc.count_shard(rp, cl, r, world, partial, per_vertex_partial=pv)
        torch.cuda.synchronize()
        parts.append(int(partial.item()))
        pv_sum += pv
    assert sum(parts) == T and (pv_np(pv_sum) == t).all()
    assert sum(1 for p in parts if p > 0) >= min(world, 2)      # work really is split


@pytest.mark.parametrize("short_max", [0, 8, 20, 32, 128])
@pytest.mark.parametrize("world", [1, 3])
@pytest.mark.parametrize("gname", ["rmat", "chung_lu"])
def test_shards_with_short_bin(gname, world, short_max):
    """Owners whose in-part entries all left HASH (SHORT bin or another rank's sources)
    keep only their out-part probe entries (regression: entry indexing must skip the
    in-list consistently in the task builder and the kernels)."""
    g = G.rmat(12, 8, seed=5) if gname == "rmat" else G.chung_lu(20000, 200000, seed=6)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    rp, cl = on_dev(g.rowptr, g.col)
    tot, pv_sum = 0, torch.zeros(g.n, dtype=torch.int64, device=DEV)
    for r in range(world):
        partial = torch.zeros(1, dtype=torch.int64, device=DEV)
        pv = torch.zeros(g.n, dtype=torch.int64, device=DEV)
        tc.count_shard(rp, cl, r, world, partial, per_vertex_partial=pv, short_max=short_max)
        torch.cuda.synchronize()
        tot += int(partial.item())
        pv_sum += pv
    assert tot == T and (pv_np(pv_sum) == t).all()


# ------------------------------------------------------------------ errors
def test_validate_rejects_bad_graphs():
    bad = [(np.array([0, 1, 2], np.uint64), np.array([1, 5], np.uint32)),     # id >= n
           (np.array([0, 2, 1], np.uint64), np.array([1, 0], np.uint32))]     # non-monotone
    for rp, cl in bad:
        with pytest.raises(tc.TCError) as e:
            gpu_count(rp, cl, validate=True)
        assert e.value.status == 2
    row, col = clean_csr(G.karate())
    with pytest.raises(tc.TCError):   # TC_CLEAN claim on asymmetric input
        gpu_count(np.array([0, 1, 1], np.uint64), np.array([1], np.uint32), clean=True,
                  sorted_rows=True, validate=True)
    assert gpu_count(row, col, clean=True, sorted_rows=True, validate=True) == 45


def _one_way_cycle(n):
    return np.arange(n + 1, dtype=np.uint64), ((np.arange(n) + 1) % n).astype(np.uint32)


def test_validate_clean_unsorted():
    """TC_CLEAN | TC_VALIDATE without TC_SORTED checks symmetry and duplicates too."""
    rp, cl = _one_way_cycle(64)                       # every arc lacks its reverse
    with pytest.raises(tc.TCError) as e:
        gpu_count(rp, cl, clean=True, validate=True)
    assert e.value.status == 2 and "reverse" in str(e.value)
    row, col = clean_csr(G.karate())
    dup_col = np.insert(col, 1, col[0])               # row 0: its first arc twice
    dup_row = row.copy()
    dup_row[1:] += 1
    with pytest.raises(tc.TCError) as e:
        gpu_count(dup_row, dup_col, clean=True, validate=True)
    assert e.value.status == 2 and "duplicate" in str(e.value)
    rng = np.random.default_rng(3)                    # shuffled rows, valid: accepted
    srow, scol = row.copy(), col.copy()
    for u in range(len(row) - 1):
        rng.shuffle(scol[row[u]:row[u + 1]])
    assert gpu_count(srow, scol, clean=True, validate=True) == 45


@pytest.mark.parametrize("n", [8, 1000, 70_000])
def test_false_clean_claim_is_caught(n):
    """Without TC_VALIDATE a false TC_CLEAN claim (one-way cycle: n-1 arcs pass the rank
    filter, the buffers hold n/2 + 1) must not write out of bounds: TC_EGRAPH."""
    rp, cl = _one_way_cycle(n)
    with pytest.raises(tc.TCError) as e:
        gpu_count(rp, cl, clean=True, tiny_max_n=0, lowdeg_max=0)   # (the one-kernel path symmetrises anyway)
    assert e.value.status == 2
    assert gpu_count(*clean_csr(G.karate()), clean=True) == 45   # the device is still sane


# ------------------------------------------------------------------ full-size configurations
def test_config_chung_lu_full():
    g = G.chung_lu()
    T = O.count(g.n, g.rowptr, g.col)
    assert gpu_count(g.rowptr, g.col) == T


def test_config_road_full():
    g = G.road_mesh()
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    got, pv = gpu_count(g.rowptr, g.col, per_vertex=True)
    assert got == T and (pv_np(pv) == t).all()


def test_config_clique_union_full():
    g = G.clique_union()
    T = O.count(g.n, g.rowptr, g.col)
    assert gpu_count(g.rowptr, g.col) == T


def test_config_rmat21_full():
    """BASELINE configs[1]: R-MAT s21 ef16, the bench workload, in the bench's launch config."""
    g = G.rmat(21, 16)
    T = O.count(g.n, g.rowptr, g.col)
    got, pv = gpu_count(g.rowptr, g.col, per_vertex=True)
    assert got == T
    assert gpu_count(g.rowptr, g.col) == T
    # sampled per-vertex counts by definition (edges among N(v))
    row, col = clean_csr(g)
    pvh = pv_np(pv)
    rng = np.random.default_rng(0)
    deg = np.diff(row)
    sample = np.concatenate([rng.integers(0, g.n, 300), np.argsort(deg)[-20:]])
    for v in sample:
        assert int(pvh[v]) == O.vertex_triangles(g.n, row, col, int(v)), v
    assert int(pvh.sum()) == 3 * T


def test_large_closed_forms():
    g = G.complete(3000)                       # T = C(3000,3) > 2^32: uint64 totals
    assert gpu_count(g.rowptr, g.col) == math.comb(3000, 3)
    g = G.kron_power(G.karate(), 3)
    assert gpu_count(g.rowptr, g.col) == 3_280_500
    g = G.triangulated_grid(1000, 1000)
    assert gpu_count(g.rowptr, g.col) == 2 * 999 * 999


def test_kronecker_exact_pins():
    """Closed forms at scale (no oracle): T(B (x) C) = 6 T(B) T(C), t = 2 t_B t_C."""
    k3 = G.kron_power(G.karate(), 3)
    g = G.kron(k3, G.fig_mm())                               # n = 275,128, m = 37,964,160
    got, pv = gpu_count(g.rowptr, g.col, per_vertex=True)
    assert got == 6 * 3_280_500 * 3 == 59_049_000
    # per-vertex closed form: t(u1, u2) = 2 t_{k3}(u1) t_{fig}(u2), with t_{k3} from the
    # closed form again (karate^3 = karate (x) karate^2)
    tk = np.array([18, 12, 11, 10, 2, 3, 3, 6, 5, 0, 2, 0, 1, 6, 1, 1, 1, 1, 1, 1, 1, 1, 1, 4,
                   1, 1, 1, 1, 1, 4, 3, 3, 13, 15], dtype=np.uint64)      # karate (golden)
    tk2 = 2 * np.outer(tk, tk).reshape(-1)
    tk3 = 2 * np.outer(tk, tk2).reshape(-1)
    tfig = np.array([2, 1, 0, 1, 2, 3, 0], dtype=np.uint64)
    assert (pv_np(pv) == 2 * np.outer(tk3, tfig).reshape(-1)).all()


def test_karate_fourth_power():
    """karate^(x)4: n = 1,336,336, m = 296,120,448, T = 6^3 * 45^4 = 885,735,000 (s24-sized)."""
    g = G.kron_power(G.karate(), 4)
    got, st = gpu_count(g.rowptr, g.col, with_stats=True)
    assert st["m_undirected"] == 2 ** 3 * 78 ** 4 == 296_120_448
    assert got == 6 ** 3 * 45 ** 4 == 885_735_000


# ------------------------------------------------------------------ NEXT-1: clustering
# Bar (R14): every local c(v), the wedge count, T and the transitivity are
# bit-exact (each c(v) and 3T/wedges is one correctly rounded fp64 division of exact
# integers on both sides); the average is an fp64 sum in a different order, so it is
# compared within the recursive-summation bound n * 2^-53 * sum_v c(v) (c(v) >= 0).
def check_clustering(g, **kw):
    cc_o, s_o = O.clustering(g.n, g.rowptr, g.col)
    rp, cl = on_dev(g.rowptr, g.col)
    cc, s, t = tc.clustering(rp, cl, per_vertex=True, **kw)
    torch.cuda.synchronize()
    _, t_o = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    assert (cc.cpu().numpy() == cc_o).all(), g.name
    assert (pv_np(t) == t_o).all(), g.name
    assert s["triangles"] == s_o["triangles"] and s["wedges"] == s_o["wedges"], g.name
    assert s["transitivity"] == s_o["transitivity"], g.name
    bound = max(g.n, 1) * 2.0 ** -53 * s_o["avg_clustering"] * max(g.n, 1)
    assert abs(s["avg_clustering"] * g.n - s_o["avg_clustering"] * g.n) <= bound + 1e-300, g.name
    return cc, s


def test_clustering_fixtures():
    cc, s = check_clustering(G.karate())
    assert s["triangles"] == 45 and s["wedges"] == 528 and s["transitivity"] == 135 / 528
    assert round(s["avg_clustering"], 5) == 0.57064
    cc, s = check_clustering(G.complete(40))
    assert (cc.cpu().numpy() == 1.0).all() and s["transitivity"] == 1.0
    for g in (G.wheel(9), G.friendship(7), G.complete_multipartite([2, 3, 4]), G.star(12),
              G.random_tree(300, seed=2), G.fig_mm()):
        check_clustering(g)


@pytest.mark.parametrize("gname", ["rmat12", "rmat16_dirty", "chung_lu_small", "clique_small", "road_small"])
def test_clustering_generators(gname):
    g = {"rmat12": lambda: G.rmat(12, 16, seed=4),
         "rmat16_dirty": lambda: G.dirty(G.rmat(16, 8, seed=9), seed=1),
         "chung_lu_small": lambda: G.chung_lu(20000, 200000, seed=6),
         "clique_small": lambda: G.clique_union(5000, 8000, seed=3),
         "road_small": lambda: G.road_mesh(200, 200, seed=2)}[gname]()
    check_clustering(g)


def test_clustering_host_clean_and_variants():
    g = G.rmat(13, 16, seed=8)
    cc_o, s_o = O.clustering(g.n, g.rowptr, g.col)
    cc, s = tc.clustering(g.rowptr, g.col)                       # host pointers
    assert (cc == cc_o).all() and s["wedges"] == s_o["wedges"]
    crow, ccol = O.clean(g.n, g.rowptr, g.col)                   # TC_CLEAN input
    rp, cl = on_dev(crow, ccol)
    for v in VARIANTS:
        cc, s = tc.clustering(rp, cl, clean=True, force_variant=v)
        torch.cuda.synchronize()
        assert (cc.cpu().numpy() == cc_o).all() and s["transitivity"] == s_o["transitivity"], v
    e = G.from_edges(5, np.zeros((0, 2), np.int64))              # no edges: all zero
    cc, s = tc.clustering(e.rowptr, e.col)
    assert (cc == 0).all() and s == dict(triangles=0, wedges=0, transitivity=0.0, avg_clustering=0.0)


def test_clustering_rmat21_full():
    """Bench workload (R-MAT s21 ef16, raw arcs): every c(v) bit-exact."""
    g = G.rmat(21, 16)
    check_clustering(g)


def test_hash_owners_beyond_bitmap_range():
    """CTA hash owners whose rank span exceeds the 2^17-bit bitmap (n > 2^17), including
    an owner with more elements than one hash chunk (TC_ID_ORDER puts a 1500-clique on
    low ids: owner 0 has d+ = 1499 > kHashChunk)."""
    n = 300_000
    e = [(i, j) for i in range(1500) for j in range(i + 1, 1500)]        # K_1500 on 0..1499
    top = list(range(290_000, 290_100))
    e += [(10, v) for v in top] + [(a, b) for i, a in enumerate(top) for b in top[i + 1:]]
    g = G.from_edges(n, e)
    want = math.comb(1500, 3) + math.comb(101, 3)
    for kw in (dict(id_order=True), dict(id_order=True, hub_min_dplus=2), dict()):
        assert gpu_count(g.rowptr, g.col, **kw) == want, kw
    # R-MAT with many CTA owners below the top window (hub_min_dplus small)
    r = G.rmat(18, 16, seed=3)
    T = O.count(r.n, r.rowptr, r.col)
    for kw in (dict(hub_min_dplus=8), dict(hub_min_dplus=16, id_order=True), dict()):
        assert gpu_count(r.rowptr, r.col, **kw) == T, kw


# ------------------------------------------------------------------ workspace hook (§8(b))
def test_workspace_hook_counts_every_byte():
    """tc_options.alloc / free: every workspace block goes through the caller's hook, on the
    call's stream, and every block is freed before the call returns."""
    g = G.rmat(14, 16, seed=4)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    rp, cl = on_dev(g.rowptr, g.col)
    stream = torch.cuda.current_stream().cuda_stream
    live, log = {}, []

    def alloc(size, s):
        assert (s or 0) == stream          # ctypes passes the NULL (legacy) stream as None
        p = torch._C._cuda_cudaCachingAllocator_raw_alloc(size, s or 0)
        live[p] = size
        log.append(size)
        return p

    def free(p, s):
        assert (s or 0) == stream and p in live
        del live[p]
        torch._C._cuda_cudaCachingAllocator_raw_delete(p)

    for kw in [dict(), dict(per_vertex=True), dict(force_variant=tc.VARIANT_MERGE),
               dict(prune=True, prune_rounds=2)]:
        out = tc.count_ex(rp, cl, allocator=(alloc, free), **kw)
        torch.cuda.synchronize()
        got = out[0] if isinstance(out, tuple) else out
        assert got == T, kw
        if kw.get("per_vertex"):
            assert (pv_np(out[1]) == t).all()
        assert not live, f"{len(live)} workspace blocks not freed ({kw})"
    assert len(log) > 10 and sum(log) > 16 * g.arcs   # the 64-bit sort keys alone are 16 B/arc
    n_before = len(log)
    _, _, sup = tc.edge_support(rp, cl, allocator=(alloc, free))
    T2, tri = tc.enumerate_triangles(rp, cl, allocator=(alloc, free))
    _, clus = tc.clustering(rp, cl, allocator=(alloc, free))
    torch.cuda.synchronize()
    assert T2 == T and clus["triangles"] == T and int(sup.to(torch.int64).sum()) == 3 * T
    assert not live and len(log) > n_before


def test_workspace_hook_failure_is_enomem():
    g = G.rmat(10, 16, seed=4)
    rp, cl = on_dev(g.rowptr, g.col)
    with pytest.raises(tc.TCError) as e:
        tc.count_ex(rp, cl, allocator=(lambda size, s: 0, lambda p, s: None))
    assert e.value.status == 3
    assert tc.count_ex(rp, cl) == O.count(g.n, g.rowptr, g.col)   # next call is fine


def test_library_pool_and_trim():
    """Without a hook the library's own pool is used; the process default pool is untouched."""
    g = G.rmat(12, 16, seed=4)
    T = O.count(g.n, g.rowptr, g.col)
    rp, cl = on_dev(g.rowptr, g.col)
    assert tc.count_ex(rp, cl, allocator="library") == T
    assert tc.count_ex(rp, cl, allocator="library", keep_workspace=False) == T
    tc.trim_workspace()
    assert tc.count_ex(rp, cl, allocator="library") == T


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two devices")
def test_wrong_device_pointer_rejected():
    g = G.karate()
    rp = torch.from_numpy(g.rowptr.view(np.int64)).to("cuda:1")
    cl = torch.from_numpy(g.col.view(np.int32)).to("cuda:1")
    assert tc.count_ex(rp, cl) == 45            # the binding makes cuda:1 current
    lib = tc._load()
    total = __import__("ctypes").c_uint64()
    with torch.cuda.device(0):
        assert lib.tc_count_ex(g.n, g.arcs, rp.data_ptr(), cl.data_ptr(), 0, None,
                               __import__("ctypes").addressof(total), None, None) == 1


# ------------------------------------------------------------------ dense core (core.cu)
CORE_GRAPHS = {
    "karate": G.karate,                                   # n < 128: the whole graph is the core
    "K700": lambda: G.complete(700),
    "rmat14": lambda: G.rmat(14, 16, seed=21),
    "rmat17": lambda: G.rmat(17, 16, seed=22),             # n > the 16384-id core
    "clique": lambda: G.clique_union(60_000, 90_000),
    "gnp": lambda: G.gnp(3000, 0.05, 7),
    "kron2": lambda: G.kron_power(G.karate(), 2),
}


@pytest.mark.parametrize("name", sorted(CORE_GRAPHS))
def test_core_path_counts(name):
    """Plain counts under AUTO route dense-core edges to the bitmap-AND path (core.cu); the
    total must equal the oracle, and the core path must have run where the graph has a core."""
    g = CORE_GRAPHS[name]()
    T = O.count(g.n, g.rowptr, g.col)
    got, st = gpu_count(g.rowptr, g.col, with_stats=True, tiny_max_n=0, lowdeg_max=0)
    assert got == T
    if name != "karate":
        assert st["core_edges"] > 0 and st["core_words"] > 0, st
    # the per-vertex call does not use the core path: same total, zero core edges
    got2, _, st2 = gpu_count(g.rowptr, g.col, per_vertex=True, with_stats=True, tiny_max_n=0, lowdeg_max=0)
    assert got2 == T and st2["core_edges"] == 0
    # a forced variant disables it too
    got3, st3 = gpu_count(g.rowptr, g.col, force_variant=tc.VARIANT_HASH, with_stats=True)
    assert got3 == T and st3["core_edges"] == 0
    # shards: core edges split by edge range, HASH by owner
    rp, cl = on_dev(g.rowptr, g.col)
    for world in (2, 3, 8):
        tot = 0
        for r in range(world):
            p = torch.zeros(1, dtype=torch.int64, device=DEV)
            tc.count_shard(rp, cl, r, world, p)
            tot += int(p.item())
        assert tot == T, world


# ------------------------------------------------------------------ tiny graphs (tiny.cu)
TINY_GRAPHS = {
    "fig_mm": G.fig_mm, "karate": G.karate, "K20": lambda: G.complete(20),
    "K1024": lambda: G.complete(1024),                               # the size limit
    "gnp1000": lambda: G.dirty(G.gnp(1000, 0.1, 3), seed=4),          # duplicates, loops, reversed
    "rmat10": lambda: G.rmat(10, 16, seed=5),
    "wheel": lambda: G.wheel(600), "star": lambda: G.star(900), "path": lambda: G.path(1000),
    "single": lambda: G.from_edges(2, [(0, 1)]),
}


@pytest.mark.parametrize("name", sorted(TINY_GRAPHS))
def test_tiny_path(name):
    """n <= 1024: the one-kernel path (tiny.cu) against the oracle, total and every t(v), and
    against the general pipeline (tiny_max_n = 0) on the same input."""
    g = TINY_GRAPHS[name]()
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    got, pv, st = gpu_count(g.rowptr, g.col, per_vertex=True, with_stats=True)
    assert got == T and (pv_np(pv) == t).all()
    assert st["kernel_launches"] == 1
    assert st["m_undirected"] == O.count(g.n, g.rowptr, g.col, with_stats=True)[1]["m"]
    assert gpu_count(g.rowptr, g.col) == T
    got2, pv2 = gpu_count(g.rowptr, g.col, per_vertex=True, tiny_max_n=0, lowdeg_max=0)
    assert got2 == T and (pv_np(pv2) == t).all()
    rp, cl = on_dev(g.rowptr, g.col)
    tot = 0
    for r in range(3):            # shards: rank 0 takes the whole tiny graph
        p = torch.zeros(1, dtype=torch.int64, device=DEV)
        tc.count_shard(rp, cl, r, 3, p)
        tot += int(p.item())
    assert tot == T
    h = tc.count_ex(g.rowptr, g.col, per_vertex=True)               # host pointers
    assert h[0] == T and (h[1] == t).all()


# ------------------------------------------------------------------ sharded a1 (multi-GPU)
@pytest.mark.parametrize("name", ["rmat14", "dirty_gnp", "clique", "road"])
def test_sharded_clean_then_count(name):
    """tc_clean_shard on every rank + the exchange (degree sum, edge concatenation), emulated
    on one GPU, then tc_count_edges_shard per rank: the gathered edges are exactly the
    oracle's clean edge set, the summed degrees its degrees, and the partial counts (and
    per-vertex partials) sum to the oracle's."""
    g = {"rmat14": lambda: G.rmat(14, 16, seed=12), "dirty_gnp": lambda: G.dirty(G.gnp(3000, 0.01, 5), seed=6),
         "clique": lambda: G.clique_union(30_000, 40_000), "road": lambda: G.road_mesh(300, 200, seed=3)}[name]()
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    b = max(1, (g.n - 1).bit_length())
    src = np.repeat(np.arange(g.n, dtype=np.uint64), np.diff(crow).astype(np.int64))
    want_keys = np.sort(((src << np.uint64(b)) | ccol.astype(np.uint64))[src < ccol.astype(np.uint64)])
    want_deg = np.diff(crow).astype(np.int64)
    rp, cl = on_dev(g.rowptr, g.col)
    for world in (1, 2, 3, 8):
        parts = [tc.clean_shard(rp, cl, r, world) for r in range(world)]
        edges = torch.cat([e for e, _ in parts])
        deg = sum(d.to(torch.int64) for _, d in parts).to(torch.int32)
        got_keys = np.sort(edges.cpu().numpy().view(np.uint64))
        assert (got_keys == want_keys).all(), world
        assert (deg.cpu().numpy() == want_deg).all(), world
        tot, pv_sum = 0, torch.zeros(g.n, dtype=torch.int64, device=DEV)
        for r in range(world):
            p = torch.zeros(1, dtype=torch.int64, device=DEV)
            pv = torch.zeros(g.n, dtype=torch.int64, device=DEV)
            tc.count_edges_shard(g.n, edges, deg, r, world, p, per_vertex_partial=pv)
            tot += int(p.item())
            pv_sum += pv
        torch.cuda.synchronize()
        assert tot == T and (pv_np(pv_sum) == t).all(), world
