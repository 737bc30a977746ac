"""Seeded synthetic graph inputs, shared by tests, the oracle side and bench.py.

This module draws arcs and packages them as a CSR grouped by source.  It holds
none of the triangle-counting method's arithmetic: no cleaning, no degree
order, no intersection.  Outputs are RAW arc lists (duplicates, self-loops and
one-directional arcs included) -- cleaning them is the method's step a1.

Large generators are in ``graphgen/gen.c`` (counter-based RNG, OpenMP; the
result does not depend on the thread count).  Small closed-form families are
plain numpy.  Input recipes: DESIGN.md "Inputs" / SURVEY.md §8(d).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libgraphgen.so")
_lib = None
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.run(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11", "-Wall",
                        "-o", _LIB, _SRC, "-lm"], check=True)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        vp, u64, u32, dbl = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double
        lib.gen_rmat.argtypes = [u32, u64, u64, vp, vp]
        lib.gen_rmat.restype = None
        lib.gen_chung_lu.argtypes = [u64, u64, dbl, dbl, u64, vp, vp]
        lib.gen_chung_lu.restype = ctypes.c_int
        lib.gen_road_mesh.argtypes = [u64, u64, dbl, dbl, u64, vp, vp, u64]
        lib.gen_road_mesh.restype = ctypes.c_int64
        lib.gen_clique_union_sizes.argtypes = [u64, u32, u32, dbl, u64, vp]
        lib.gen_clique_union_sizes.restype = u64
        lib.gen_clique_union_fill.argtypes = [u64, u64, vp, dbl, u64, vp, vp]
        lib.gen_clique_union_fill.restype = ctypes.c_int
        lib.gen_kron.argtypes = [u64, u64, vp, vp, u64, vp, vp, vp, vp]
        lib.gen_kron.restype = None
        lib.gen_arcs_to_csr.argtypes = [u64, u64, vp, vp, vp, vp]
        lib.gen_arcs_to_csr.restype = ctypes.c_int
        lib.gen_draw.argtypes = [u64, u64, u64]
        lib.gen_draw.restype = u64
        lib.gen_perm.argtypes = [u64, u64, u64]
        lib.gen_perm.restype = u64
        _lib = lib
    return _lib


@dataclasses.dataclass
class Graph:
    """A raw input graph: n vertices, arcs u -> col[k] for rowptr[u] <= k < rowptr[u+1]."""
    n: int
    rowptr: np.ndarray  # uint64[n+1]
    col: np.ndarray     # uint32[M]
    name: str = ""

    @property
    def arcs(self) -> int:
        return int(self.rowptr[-1]) if len(self.rowptr) else 0

    def arc_list(self):
        src = np.repeat(np.arange(self.n, dtype=np.uint32), np.diff(self.rowptr).astype(np.int64))
        return src, self.col.copy()


def from_arcs(n: int, src, dst, name: str = "") -> Graph:
    """Package arcs (src[i] -> dst[i]) as a CSR grouped by source, draw order kept."""
    src = np.ascontiguousarray(src, dtype=np.uint32)
    dst = np.ascontiguousarray(dst, dtype=np.uint32)
    if src.shape != dst.shape:
        raise ValueError("src/dst length mismatch")
    rowptr = np.zeros(n + 1, dtype=np.uint64)
    col = np.zeros(max(1, src.size), dtype=np.uint32)
    r = _load().gen_arcs_to_csr(n, src.size, src.ctypes.data, dst.ctypes.data,
                                rowptr.ctypes.data, col.ctypes.data)
    if r != 0:
        raise ValueError("arc endpoint >= n")
    return Graph(n, rowptr, col[:src.size].copy(), name)


def from_edges(n: int, edges, name: str = "") -> Graph:
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    return from_arcs(n, e[:, 0], e[:, 1], name)


def symmetric_arcs(g: Graph) -> Graph:
    """Add the reverse of every arc (a format change only: duplicates stay)."""
    s, d = g.arc_list()
    return from_arcs(g.n, np.concatenate([s, d]), np.concatenate([d, s]), g.name)


# ---------------------------------------------------------------- fixtures
# Zachary karate club (34 vertices, 78 edges): each vertex followed by its
# higher-id neighbours.
_KARATE = {
    0: [1, 2, 3, 4, 5, 6, 7, 8, 10, 11, 12, 13, 17, 19, 21, 31],
    1: [2, 3, 7, 13, 17, 19, 21, 30], 2: [3, 7, 8, 9, 13, 27, 28, 32], 3: [7, 12, 13],
    4: [6, 10], 5: [6, 10, 16], 6: [16], 8: [30, 32, 33], 9: [33], 13: [33], 14: [32, 33],
    15: [32, 33], 18: [32, 33], 19: [33], 20: [32, 33], 22: [32, 33],
    23: [25, 27, 29, 32, 33], 24: [25, 27, 31], 25: [31], 26: [29, 33], 27: [33],
    28: [31, 33], 29: [32, 33], 30: [32, 33], 31: [32, 33], 32: [33],
}


def karate_edges():
    return [(u, v) for u, vs in _KARATE.items() for v in vs]


def karate() -> Graph:
    return from_edges(34, karate_edges(), "karate")


def fig_mm_edges():
    """The 7-vertex example graph, read off matrix A of Fig. mm."""
    A = np.array([[0, 1, 0, 0, 1, 1, 0], [1, 0, 1, 0, 0, 1, 0], [0, 1, 0, 1, 0, 0, 1],
                  [0, 0, 1, 0, 1, 1, 0], [1, 0, 0, 1, 0, 1, 0], [1, 1, 0, 1, 1, 0, 0],
                  [0, 0, 1, 0, 0, 0, 0]])
    return [(i, j) for i in range(7) for j in range(i + 1, 7) if A[i, j]]


def fig_mm() -> Graph:
    return from_edges(7, fig_mm_edges(), "fig_mm")


def complete(n: int) -> Graph:
    return from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)], f"K{n}")


def wheel(n: int) -> Graph:
    """n vertices: hub 0 plus an (n-1)-cycle on 1..n-1."""
    rim = list(range(1, n))
    e = [(0, v) for v in rim] + [(rim[i], rim[(i + 1) % len(rim)]) for i in range(len(rim))]
    return from_edges(n, e, f"W{n}")


def cycle(n: int) -> Graph:
    return from_edges(n, [(i, (i + 1) % n) for i in range(n)], f"C{n}")


def path(n: int) -> Graph:
    return from_edges(n, [(i, i + 1) for i in range(n - 1)], f"P{n}")


def star(k: int) -> Graph:
    return from_edges(k + 1, [(0, i) for i in range(1, k + 1)], f"S{k}")


def random_tree(n: int, seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    e = [(i, int(rng.integers(0, i))) for i in range(1, n)]
    return from_edges(n, e, f"tree{n}")


def random_bipartite(a: int, b: int, p: float, seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    mask = rng.random((a, b)) < p
    ii, jj = np.nonzero(mask)
    return from_edges(a + b, np.stack([ii, jj + a], 1), f"bip{a}x{b}")


def complete_multipartite(sizes) -> Graph:
    part = np.repeat(np.arange(len(sizes)), sizes)
    n = int(sum(sizes))
    ii, jj = np.triu_indices(n, 1)
    keep = part[ii] != part[jj]
    return from_edges(n, np.stack([ii[keep], jj[keep]], 1), f"K{tuple(sizes)}")


def friendship(k: int) -> Graph:
    """k triangles sharing vertex 0."""
    e = []
    for t in range(k):
        a, b = 1 + 2 * t, 2 + 2 * t
        e += [(0, a), (0, b), (a, b)]
    return from_edges(2 * k + 1, e, f"F{k}")


def windmill(k: int, s: int) -> Graph:
    """k copies of K_s sharing hub 0."""
    e = []
    for c in range(k):
        vs = [0] + [1 + c * (s - 1) + i for i in range(s - 1)]
        e += [(vs[i], vs[j]) for i in range(s) for j in range(i + 1, s)]
    return from_edges(1 + k * (s - 1), e, f"Wd{k},{s}")


def gnp(n: int, p: float, seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    ii, jj = np.triu_indices(n, 1)
    keep = rng.random(ii.size) < p
    return from_edges(n, np.stack([ii[keep], jj[keep]], 1), f"G({n},{p})")


def disjoint_union(*gs: Graph) -> Graph:
    srcs, dsts, off = [], [], 0
    for g in gs:
        s, d = g.arc_list()
        srcs.append(s.astype(np.int64) + off)
        dsts.append(d.astype(np.int64) + off)
        off += g.n
    return from_arcs(off, np.concatenate(srcs), np.concatenate(dsts), "union")


# ---------------------------------------------------------------- perturbations
def dirty(g: Graph, seed: int, dup: float = 0.3, loops: int = 5, reverse: float = 0.5,
          shuffle: bool = True) -> Graph:
    """Same simple graph, messier arcs: duplicates, self-loops, flipped arcs, shuffled rows."""
    rng = np.random.default_rng(seed)
    s, d = g.arc_list()
    s = s.astype(np.int64)
    d = d.astype(np.int64)
    flip = rng.random(s.size) < reverse
    s2 = np.where(flip, d, s)
    d2 = np.where(flip, s, d)
    k = rng.random(s.size) < dup
    s3 = np.concatenate([s2, d[k]])
    d3 = np.concatenate([d2, s[k]])
    if g.n > 0 and loops:
        lv = rng.integers(0, g.n, loops)
        s3 = np.concatenate([s3, lv])
        d3 = np.concatenate([d3, lv])
    if shuffle:
        p = rng.permutation(s3.size)
        s3, d3 = s3[p], d3[p]
    return from_arcs(g.n, s3, d3, g.name + "+dirty")


def relabel(g: Graph, seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    p = rng.permutation(g.n)
    s, d = g.arc_list()
    return from_arcs(g.n, p[s], p[d], g.name + "+relabel")


# ---------------------------------------------------------------- large generators
def rmat(scale: int, edge_factor: int = 16, seed: int | None = None) -> Graph:
    """Graph500 R-MAT (A,B,C,D = .57,.19,.19,.05), edge_factor * 2^scale raw arcs."""
    lib = _load()
    seed = scale if seed is None else seed
    n = 1 << scale
    npairs = edge_factor * n
    src = np.empty(npairs, dtype=np.uint32)
    dst = np.empty(npairs, dtype=np.uint32)
    lib.gen_rmat(scale, npairs, seed, src.ctypes.data, dst.ctypes.data)
    g = from_arcs(n, src, dst, f"rmat-s{scale}-ef{edge_factor}")
    return g


def chung_lu(n: int = 4_847_571, npairs: int = 68_993_773, alpha: float = 0.7,
             i0: float = 76.865, seed: int = 7) -> Graph:
    """Chung-Lu power-law graph with a LiveJournal-like degree sequence."""
    lib = _load()
    src = np.empty(npairs, dtype=np.uint32)
    dst = np.empty(npairs, dtype=np.uint32)
    if lib.gen_chung_lu(n, npairs, alpha, i0, seed, src.ctypes.data, dst.ctypes.data) != 0:
        raise MemoryError("gen_chung_lu")
    return from_arcs(n, src, dst, f"chung-lu-n{n}")


def road_mesh(W: int = 3753, H: int = 3753, p: float = 0.56, q: float = 0.0825,
              seed: int = 11) -> Graph:
    """Road-network-like planar mesh, max degree <= 8."""
    lib = _load()
    cap = 3 * W * H
    src = np.empty(cap, dtype=np.uint32)
    dst = np.empty(cap, dtype=np.uint32)
    k = lib.gen_road_mesh(W, H, p, q, seed, src.ctypes.data, dst.ctypes.data, cap)
    if k < 0:
        raise RuntimeError("gen_road_mesh capacity")
    return from_arcs(W * H, src[:k], dst[:k], f"mesh{W}x{H}")


def triangulated_grid(W: int, H: int, seed: int = 1) -> Graph:
    """Every lattice edge plus one diagonal per cell: T = 2(W-1)(H-1)."""
    return road_mesh(W, H, 1.0, 1.0, seed)


def clique_union(n: int = 540_486, groups: int = 850_000, smin: int = 2, smax: int = 64,
                 gamma: float = 2.5, beta: float = 0.35, seed: int = 5) -> Graph:
    """Union of cliques on power-law-chosen members (co-author-like)."""
    lib = _load()
    sizes = np.empty(groups, dtype=np.uint32)
    tot = lib.gen_clique_union_sizes(groups, smin, smax, gamma, seed, sizes.ctypes.data)
    src = np.empty(max(1, tot), dtype=np.uint32)
    dst = np.empty(max(1, tot), dtype=np.uint32)
    if lib.gen_clique_union_fill(n, groups, sizes.ctypes.data, beta, seed,
                                 src.ctypes.data, dst.ctypes.data) != 0:
        raise MemoryError("gen_clique_union_fill")
    return from_arcs(n, src[:tot], dst[:tot], f"clique-union-n{n}")


def _kron_arcs(sa, da, nb, sb, db):
    N = sa.size * sb.size
    src = np.empty(max(1, N), dtype=np.uint32)
    dst = np.empty(max(1, N), dtype=np.uint32)
    _load().gen_kron(nb, sa.size, sa.ctypes.data, da.ctypes.data, sb.size, sb.ctypes.data,
                     db.ctypes.data, src.ctypes.data, dst.ctypes.data)
    return src[:N], dst[:N]


def kron(a: Graph, b: Graph) -> Graph:
    """Kronecker (tensor) product of the symmetrised arc sets of a and b."""
    sa, da = symmetric_arcs(a).arc_list()
    sb, db = symmetric_arcs(b).arc_list()
    s, d = _kron_arcs(sa, da, b.n, sb, db)
    return from_arcs(a.n * b.n, s, d, f"({a.name}x{b.name})")


def kron_power(base: Graph, k: int) -> Graph:
    """base^{(x)k}: arcs are (sym arcs of base)^k, each undirected edge in both directions."""
    sb, db = symmetric_arcs(base).arc_list()
    s, d, n = sb, db, base.n
    for _ in range(k - 1):
        s, d = _kron_arcs(s, d, base.n, sb, db)
        n *= base.n
    return from_arcs(n, s, d, f"{base.name}^{k}")
