"""CPU oracle for exact triangle counting -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product package ``paper_1804_06926_b200`` never imports it and shares no
code with it.

The arithmetic lives in ``oracle/tc_oracle.c`` (plain C, OpenMP over source
vertices only); this module is argument marshalling over ctypes plus the
build step.  Every function cites the PAPER.md passage it follows in the C
file's comments.

Parity status: every function here is pinned by ``tests/test_oracle_pins.py``
(paper worked example, closed forms, brute force, trace(A^3)/6, Kronecker
products); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)


# TC_ORACLE_SANITIZE=1: build and load an AddressSanitizer + UBSan build instead (run the
# Python process with LD_PRELOAD=$(gcc -print-file-name=libasan.so), see
# scripts/oracle_sanitize.sh); any report aborts the process.
_SANITIZE = os.environ.get("TC_ORACLE_SANITIZE") == "1"
if _SANITIZE:
    _LIB = os.path.join(_HERE, "liboracle_asan.so")


def build(force: bool = False) -> str:
    """Compile tc_oracle.c into liboracle.so (gcc, -O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=c11", "-Wall",
               "-o", _LIB, _SRC]
        if _SANITIZE:
            cmd[1:1] = ["-g", "-fsanitize=address,undefined", "-fno-omit-frame-pointer",
                        "-fno-sanitize-recover=undefined"]
        subprocess.run(cmd, check=True)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_clean.restype = ctypes.c_int64
        lib.oracle_clean.argtypes = [ctypes.c_uint64, _u64p, _u32p, _u64p, _u32p]
        lib.oracle_orient.restype = ctypes.c_int64
        lib.oracle_orient.argtypes = [ctypes.c_uint64, _u64p, _u32p, _u64p, _u32p]
        lib.oracle_forward.restype = ctypes.c_uint64
        lib.oracle_forward.argtypes = [ctypes.c_uint64, _u64p, _u32p, ctypes.c_void_p]
        lib.oracle_count.restype = ctypes.c_int
        lib.oracle_count.argtypes = [ctypes.c_uint64, _u64p, _u32p, _u64p,
                                     ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_vertex_triangles.restype = ctypes.c_uint64
        lib.oracle_vertex_triangles.argtypes = [ctypes.c_uint64, _u64p, _u32p, ctypes.c_uint64]
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_prune.restype = ctypes.c_int64
        lib.oracle_prune.argtypes = [ctypes.c_uint64, _u64p, _u32p, ctypes.c_uint32, _u64p, _u32p,
                                     ctypes.c_void_p]
        lib.oracle_edge_support.restype = None
        lib.oracle_edge_support.argtypes = [ctypes.c_uint64, _u64p, _u32p, _u64p, _u32p, _u32p]
        lib.oracle_orient_order.restype = ctypes.c_int64
        lib.oracle_orient_order.argtypes = [ctypes.c_uint64, _u64p, _u32p, ctypes.c_int, _u64p, _u32p]
        lib.oracle_masked_spgemm.restype = ctypes.c_uint64
        lib.oracle_masked_spgemm.argtypes = [ctypes.c_uint64, _u64p, _u32p, ctypes.c_int, _u64p, _u32p,
                                             _u32p]
        lib.oracle_enumerate.restype = ctypes.c_uint64
        lib.oracle_enumerate.argtypes = [ctypes.c_uint64, _u64p, _u32p, ctypes.c_void_p,
                                         ctypes.c_uint64]
        lib.oracle_clustering.restype = None
        lib.oracle_clustering.argtypes = [ctypes.c_uint64, _u64p, _u64p, ctypes.c_uint64,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]
        _lib = lib
    return _lib


def _csr(rowptr, col):
    rowptr = np.ascontiguousarray(rowptr, dtype=np.uint64)
    col = np.ascontiguousarray(col, dtype=np.uint32)
    if col.size == 0:
        col = np.zeros(1, dtype=np.uint32)          # never read; keeps a valid pointer
    return rowptr, col


def _p64(a):
    return a.ctypes.data_as(_u64p)


def _p32(a):
    return a.ctypes.data_as(_u32p)


def clean(n: int, rowptr, col):
    """Step 1: simple undirected graph as symmetric sorted CSR."""
    lib = _load()
    rowptr, col = _csr(rowptr, col)
    out_row = np.zeros(n + 1, dtype=np.uint64)
    out_col = np.zeros(max(1, 2 * int(rowptr[n])), dtype=np.uint32)
    r = lib.oracle_clean(n, _p64(rowptr), _p32(col), _p64(out_row), _p32(out_col))
    if r < 0:
        raise ValueError(f"oracle_clean failed ({r}): arc id >= n or out of memory")
    return out_row, out_col[:r].copy()


def orient(n: int, clean_rowptr, clean_col):
    """Step 2 (Alg. 2 Form_Filtered_Edge_List): N+ lists by (deg, id)."""
    lib = _load()
    clean_rowptr, clean_col = _csr(clean_rowptr, clean_col)
    off = np.zeros(n + 1, dtype=np.uint64)
    colp = np.zeros(max(1, int(clean_rowptr[n]) // 2 + 1), dtype=np.uint32)
    m = lib.oracle_orient(n, _p64(clean_rowptr), _p32(clean_col), _p64(off), _p32(colp))
    return off, colp[:m].copy()


def forward(n: int, off_plus, col_plus, per_vertex: bool = False):
    """Steps 3+4 on an oriented CSR; returns T or (T, t)."""
    lib = _load()
    off_plus, col_plus = _csr(off_plus, col_plus)
    pv = np.zeros(max(n, 1), dtype=np.uint64) if per_vertex else None
    T = lib.oracle_forward(n, _p64(off_plus), _p32(col_plus),
                           pv.ctypes.data if pv is not None else None)
    return (int(T), pv[:n]) if per_vertex else int(T)


def count(n: int, rowptr, col, per_vertex: bool = False, with_stats: bool = False):
    """Whole oracle: T (and t(v), stats) of the simple graph the arcs define."""
    lib = _load()
    rowptr, col = _csr(rowptr, col)
    if int(rowptr[0]) != 0 or len(rowptr) != n + 1:
        raise ValueError("rowptr must have n+1 entries starting at 0")
    total = np.zeros(1, dtype=np.uint64)
    pv = np.zeros(max(n, 1), dtype=np.uint64) if per_vertex else None
    st = np.zeros(8, dtype=np.uint64)
    r = lib.oracle_count(n, _p64(rowptr), _p32(col), _p64(total),
                         pv.ctypes.data if pv is not None else None, st.ctypes.data)
    if r != 0:
        raise ValueError(f"oracle_count failed ({r})")
    out = [int(total[0])]
    if per_vertex:
        out.append(pv[:n])
    if with_stats:
        out.append(dict(m=int(st[0]), W=int(st[1]), SSD=int(st[2]), sum_dminus_dplus=int(st[3]),
                        max_dplus=int(st[4]), max_deg=int(st[5]), wedges=int(st[6])))
    return out[0] if len(out) == 1 else tuple(out)


def vertex_triangles(n: int, clean_rowptr, clean_col, v: int) -> int:
    """t(v) by definition (edges among N(v)) on a clean symmetric sorted CSR."""
    lib = _load()
    clean_rowptr, clean_col = _csr(clean_rowptr, clean_col)
    return int(lib.oracle_vertex_triangles(n, _p64(clean_rowptr), _p32(clean_col), v))


def clustering(n: int, rowptr, col):
    """NEXT-1: (local cc[n], summary dict) of the simple graph the
    arcs define -- clean, per-vertex counts, then the definitions in tc_oracle.c."""
    lib = _load()
    crow, ccol = clean(n, rowptr, col)
    T, t = count(n, rowptr, col, per_vertex=True)
    t = np.ascontiguousarray(t, dtype=np.uint64)
    cc = np.zeros(max(n, 1), dtype=np.float64)
    w = np.zeros(1, dtype=np.uint64)
    s = np.zeros(1, dtype=np.float64)
    tr = np.zeros(1, dtype=np.float64)
    lib.oracle_clustering(n, _p64(crow), _p64(t) if n else None, T, cc.ctypes.data, w.ctypes.data,
                          s.ctypes.data, tr.ctypes.data)
    summary = dict(triangles=T, wedges=int(w[0]), transitivity=float(tr[0]),
                   avg_clustering=float(s[0]) / n if n else 0.0)
    return cc[:n], summary


def prune(n: int, clean_rowptr, clean_col, rounds: int = 0):
    """NEXT-2: delete edges with an endpoint of degree < 2, `rounds`
    times (0 = until nothing changes: the 2-core).  -> (rowptr, col, rounds executed)."""
    lib = _load()
    clean_rowptr, clean_col = _csr(clean_rowptr, clean_col)
    out_row = np.zeros(n + 1, dtype=np.uint64)
    out_col = np.zeros(max(1, int(clean_rowptr[n])), dtype=np.uint32)
    done = np.zeros(1, dtype=np.uint32)
    r = lib.oracle_prune(n, _p64(clean_rowptr), _p32(clean_col), rounds, _p64(out_row),
                         _p32(out_col), done.ctypes.data)
    if r < 0:
        raise MemoryError("oracle_prune: allocation failed")
    return out_row, out_col[:r].copy(), int(done[0])


def edge_support(n: int, clean_rowptr, clean_col, off_plus, col_plus):
    """NEXT-3: sup[e] = |N(u) cap N(v)| for every entry e = (u, col_plus[e]) of an
    oriented CSR, by merging the full rows of the clean symmetric CSR."""
    lib = _load()
    clean_rowptr, clean_col = _csr(clean_rowptr, clean_col)
    m = int(off_plus[n]) if n else 0
    off_plus, col_plus = _csr(off_plus, col_plus)
    sup = np.zeros(max(m, 1), dtype=np.uint32)
    lib.oracle_edge_support(n, _p64(clean_rowptr), _p32(clean_col), _p64(off_plus), _p32(col_plus),
                            _p32(sup))
    return sup[:m]


def enumerate_triangles(n: int, clean_rowptr, clean_col):
    """NEXT-3: all triangles as a (T, 3) uint32 array of (a<b<c), lexicographic."""
    lib = _load()
    clean_rowptr, clean_col = _csr(clean_rowptr, clean_col)
    T = int(lib.oracle_enumerate(n, _p64(clean_rowptr), _p32(clean_col), None, 0))
    out = np.zeros(max(3 * T, 3), dtype=np.uint32)
    T2 = int(lib.oracle_enumerate(n, _p64(clean_rowptr), _p32(clean_col), out.ctypes.data, T))
    assert T2 == T
    return out[:3 * T].reshape(T, 3)


def orient_order(n: int, clean_rowptr, clean_col, id_order: bool = False):
    """oracle.orient with the vertex order of Alg. 3 line 1 (degree, id) or, with id_order,
    plain ids (Fig. mm): the upper triangle U as a CSR, rows ascending."""
    lib = _load()
    clean_rowptr, clean_col = _csr(clean_rowptr, clean_col)
    off = np.zeros(n + 1, dtype=np.uint64)
    colp = np.zeros(max(1, int(clean_rowptr[n]) // 2 + 1), dtype=np.uint32)
    m = lib.oracle_orient_order(n, _p64(clean_rowptr), _p32(clean_col), int(id_order), _p64(off),
                                _p32(colp))
    return off, colp[:m].copy()


def masked_spgemm(n: int, clean_rowptr, clean_col, id_order: bool = False):
    """NEXT-4 (Alg. 3, masked per P:723-731): (off_u, col_u, C at U's entries, n=T)."""
    lib = _load()
    off, colp = orient_order(n, clean_rowptr, clean_col, id_order)
    clean_rowptr, clean_col = _csr(clean_rowptr, clean_col)
    m = int(off[n]) if n else 0
    c = np.zeros(max(m, 1), dtype=np.uint32)
    cp = colp if m else np.zeros(1, dtype=np.uint32)
    T = lib.oracle_masked_spgemm(n, _p64(clean_rowptr), _p32(clean_col), int(id_order), _p64(off),
                                 _p32(cp), _p32(c))
    return off, colp, c[:m], int(T)


def num_threads() -> int:
    return int(_load().oracle_num_threads())
