"""GPU parity of a1 (clean: symmetrize, de-duplicate, drop self-loops; Table 1 caption
P:604-606) under both sort orders of tc_options.clean_method: 0 (default, round 2) sorts the
64-bit (min, max) keys by a 24/32-bit hash only, so duplicates share a run of equal hash and
the unique step compares each key with the earlier keys of its run; 1 sorts the full
(min, max) order (round 1).  The graphs stress duplicates (every arc up to 3 times, flipped),
hubs (groups of 10^4-10^5 copies of one endpoint), long runs of isolated vertices and
self-loops.  Every case runs with tiny_max_n = 0 (small graphs take the pipeline, not the
one-kernel path).  T, every t(v) and the oriented CSR (off+, col+) must equal the oracle's
bit for bit (Alg. 2).
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


def on_dev(rowptr, col):
    return (torch.from_numpy(np.ascontiguousarray(rowptr, np.uint64).view(np.int64)).to(DEV),
            torch.from_numpy(np.ascontiguousarray(col, np.uint32).view(np.int32)).to(DEV))


def repeated(g, times, seed):
    """Every arc `times` times, each copy flipped at random, rows shuffled."""
    rng = np.random.default_rng(seed)
    s, d = g.arc_list()
    s = np.tile(s.astype(np.int64), times)
    d = np.tile(d.astype(np.int64), times)
    f = rng.random(s.size) < 0.5
    s, d = np.where(f, d, s), np.where(f, s, d)
    p = rng.permutation(s.size)
    return G.from_arcs(g.n, s[p], d[p], g.name + f"x{times}")


def star_at(n, centre, leaves, seed):
    rng = np.random.default_rng(seed)
    lv = rng.choice(np.setdiff1d(np.arange(n), [centre]), leaves, replace=False)
    return G.from_arcs(n, np.full(leaves, centre), lv, f"star@{centre}")


def sparse_isolated(n, m, seed):
    """A few edges among far-apart ids: long runs of empty groups."""
    rng = np.random.default_rng(seed)
    v = rng.choice(n, 64, replace=False)
    a, b = rng.choice(v, m), rng.choice(v, m)
    return G.from_arcs(n, a, b, "sparse")


def hub_mix(seed):
    """A dense hub block (8 hubs x 9000 arcs), a dense 300-vertex block, and background noise."""
    rng = np.random.default_rng(seed)
    n = 60000
    src = [np.repeat(np.arange(8), 9000), rng.integers(0, 300, 40000)]
    dst = [rng.integers(0, n, 72000), rng.integers(0, 300, 40000)]
    src.append(rng.integers(0, n, 100000))
    dst.append(rng.integers(0, n, 100000))
    s, d = np.concatenate(src), np.concatenate(dst)
    f = rng.random(s.size) < 0.5
    return G.from_arcs(n, np.where(f, d, s), np.where(f, s, d), "hubmix")


CASES = {
    "karate": G.karate,
    "dirty_gnp": lambda: G.dirty(G.gnp(3000, 0.01, 1), 1),
    "K300x3": lambda: repeated(G.complete(300), 3, 2),                 # 3 copies of every edge
    "star_low": lambda: repeated(star_at(9000, 0, 5000, 3), 2, 3),     # hub = min of every edge
    "star_high": lambda: repeated(star_at(9000, 8999, 5000, 4), 2, 4), # every arc is lower
    "star_huge": lambda: repeated(star_at(70000, 17, 60000, 5), 3, 5), # 180000 arcs at one hub
    "sparse": lambda: sparse_isolated(300000, 500, 6),
    "hubmix": lambda: hub_mix(7),
    "rmat14": lambda: G.rmat(14, 16, seed=14),
    "rmat16_dirty": lambda: G.dirty(G.rmat(16, 8, seed=16), 16, dup=0.5),
    "chung_lu": lambda: G.chung_lu(40000, 400000, seed=8),
    "mesh": lambda: G.road_mesh(300, 200, seed=9),
}


@pytest.mark.parametrize("method", [0, 1])
@pytest.mark.parametrize("name", sorted(CASES))
def test_clean_vs_oracle(name, method):
    g = CASES[name]()
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    rp, cl = on_dev(g.rowptr, g.col)
    got, pv = tc.count_ex(rp, cl, per_vertex=True, tiny_max_n=0, lowdeg_max=0, clean_method=method)
    torch.cuda.synchronize()
    assert got == T, (name, method, got, T)
    assert (pv.cpu().numpy().view(np.uint64) == t).all(), (name, method)
    row, col = O.clean(g.n, g.rowptr, g.col)
    want_off, want_col = O.orient(g.n, row, col)
    off, colp = tc.orient(rp, cl, tiny_max_n=0, lowdeg_max=0, clean_method=method)
    torch.cuda.synchronize()
    assert (off.cpu().numpy().view(np.uint64) == want_off).all(), (name, method)
    assert (colp.cpu().numpy().view(np.uint32) == want_col).all(), (name, method)


def test_clean_stats_match_oracle():
    g = G.dirty(G.rmat(13, 16, seed=31), 31, dup=0.4)
    T, st_o = O.count(g.n, g.rowptr, g.col, with_stats=True)
    rp, cl = on_dev(g.rowptr, g.col)
    got, st = tc.count_ex(rp, cl, with_stats=True, clean_method=0)
    assert got == T
    assert st["m_undirected"] == st_o["m"] and st["work_W"] == st_o["W"]
    assert st["max_dplus"] == st_o["max_dplus"] and st["work_stage"] == st_o["sum_dminus_dplus"]


@pytest.mark.parametrize("world", [2, 5])
def test_clean_shards(world):
    g = hub_mix(11)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    rp, cl = on_dev(g.rowptr, g.col)
    tot, pv_sum = 0, torch.zeros(g.n, dtype=torch.int64, device=DEV)
    for r in range(world):
        partial = torch.zeros(1, dtype=torch.int64, device=DEV)
        pv = torch.zeros(g.n, dtype=torch.int64, device=DEV)
        tc.count_shard(rp, cl, r, world, partial, per_vertex_partial=pv)
        torch.cuda.synchronize()
        tot += int(partial.item())
        pv_sum += pv
    assert tot == T and (pv_sum.cpu().numpy().view(np.uint64) == t).all()


def test_clean_host_pointers_and_allocator():
    g = repeated(star_at(20000, 5, 12000, 12), 2, 12)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    got, pv = tc.count_ex(g.rowptr, g.col, per_vertex=True)
    assert got == T and (pv == t).all()
    rp, cl = on_dev(g.rowptr, g.col)
    got = tc.count_ex(rp, cl, allocator="library")
    torch.cuda.synchronize()
    assert got == T
