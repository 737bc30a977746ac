"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/tc.h
declares, and rejects bad arguments before touching a device (no compute calls)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1804_06926_b200 as tc
from paper_1804_06926_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return tc._load()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "tc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tc_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert set(names) >= {"tc_count", "tc_count_ex", "tc_count_shard", "tc_orient",
                          "tc_clustering", "tc_edge_support", "tc_enumerate", "tc_masked_spgemm",
                          "tc_last_error", "tc_trim_workspace",
                          "tc_default_options", "tc_version"}
    for name in names:
        assert hasattr(lib, name), name


def test_sm100a_cubin_present():
    data = open(tc.library_path(), "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_struct_layout(lib):
    o = tc.Options()
    lib.tc_default_options(ctypes.byref(o))
    assert ctypes.sizeof(tc.Options) == 96
    assert tc.Options.alloc.offset == 32 and tc.Options.clean_method.offset == 60
    assert tc.Options.graph_cache.offset == 64 and tc.Options.lowdeg_max.offset == 68
    assert tc.Options.reserved.offset == 72
    assert o.graph_cache == 0
    assert o.tiny_max_n == 1024 and o.clean_method == 0 and o.lowdeg_max == 32
    assert o.short_max == 20 and o.skew_ratio == 0 and o.hub_min_dplus == 80
    assert o.force_variant == -1 and o.keep_workspace == 1
    assert not o.alloc and not o.free and not o.alloc_ctx
    assert o.prune_rounds == 0 and not any(o.reserved)
    assert ctypes.sizeof(tc.Stats) == 7 * 8 + 22 * 8
    assert ctypes.sizeof(tc.ClusteringSummary) == 32


def test_clustering_argument_errors(lib):
    rp = np.zeros(2, np.uint64)
    EINVAL = 1
    # TC_PER_VERTEX is implied by tc_clustering and rejected as a flag
    assert lib.tc_clustering(1, 0, rp.ctypes.data, None, tc.TC_PER_VERTEX | tc.TC_HOST_PTRS, None,
                             None, None, None, None) == EINVAL
    assert b"implied" in lib.tc_last_error()
    assert lib.tc_clustering(1, 0, None, None, tc.TC_HOST_PTRS, None, None, None, None, None) == EINVAL
    # leaf pruning would change d(v): rejected
    assert lib.tc_clustering(1, 0, rp.ctypes.data, None, tc.TC_PRUNE | tc.TC_HOST_PTRS, None,
                             None, None, None, None) == EINVAL
    assert b"TC_PRUNE" in lib.tc_last_error()


def test_arc_count_limit(lib):
    rp = np.zeros(2, np.uint64)
    total = np.zeros(1, np.uint64)
    # m >= 2^32 arcs is rejected before any pointer is read
    assert lib.tc_count_ex(1, 1 << 32, rp.ctypes.data, rp.ctypes.data, tc.TC_HOST_PTRS, None,
                           total.ctypes.data, None, None) == 1
    assert b"2^32" in lib.tc_last_error()


def test_next3_argument_errors(lib):
    rp = np.zeros(2, np.uint64)
    EINVAL = 1
    out = np.zeros(4, np.uint64)
    # edge support: outputs required, TC_PER_VERTEX rejected
    assert lib.tc_edge_support(1, 0, rp.ctypes.data, None, tc.TC_HOST_PTRS, None, None, None, None,
                               None, None) == EINVAL
    assert lib.tc_edge_support(1, 0, rp.ctypes.data, None, tc.TC_HOST_PTRS | tc.TC_PER_VERTEX, None,
                               out.ctypes.data, out.ctypes.data, out.ctypes.data, out.ctypes.data,
                               None) == EINVAL
    # enumeration: total required; triangles required when capacity > 0
    assert lib.tc_enumerate(1, 0, rp.ctypes.data, None, tc.TC_HOST_PTRS, None, None, 0, None,
                            None) == EINVAL
    assert lib.tc_enumerate(1, 0, rp.ctypes.data, None, tc.TC_HOST_PTRS, None, None, 5,
                            out.ctypes.data, None) == EINVAL
    assert b"capacity" in lib.tc_last_error()
    # masked SpGEMM: total and the value output are required
    assert lib.tc_masked_spgemm(1, 0, rp.ctypes.data, None, tc.TC_HOST_PTRS | tc.TC_ID_ORDER, None,
                                out.ctypes.data, out.ctypes.data, out.ctypes.data, out.ctypes.data,
                                None, None) == EINVAL
    assert b"total" in lib.tc_last_error()


def test_argument_errors_before_device(lib):
    rp = np.zeros(2, np.uint64)
    total = ctypes.c_uint64()
    EINVAL = 1
    # unknown flag bits
    assert lib.tc_count_ex(1, 0, rp.ctypes.data, None, 1 << 20, None, ctypes.addressof(total),
                           None, None) == EINVAL
    assert b"flag" in lib.tc_last_error()
    # n >= 2^32
    assert lib.tc_count_ex(1 << 32, 0, rp.ctypes.data, None, 0, None, ctypes.addressof(total),
                           None, None) == EINVAL
    # NULL row_offsets / NULL col with m > 0 / NULL total
    assert lib.tc_count_ex(1, 0, None, None, 0, None, ctypes.addressof(total), None, None) == EINVAL
    assert lib.tc_count_ex(1, 5, rp.ctypes.data, None, 0, None, ctypes.addressof(total), None,
                           None) == EINVAL
    assert lib.tc_count_ex(1, 0, rp.ctypes.data, None, 0, None, None, None, None) == EINVAL
    # per-vertex requested without an output; TC_SORTED without TC_CLEAN
    assert lib.tc_count_ex(1, 0, rp.ctypes.data, None, tc.TC_PER_VERTEX, None,
                           ctypes.addressof(total), None, None) == EINVAL
    assert lib.tc_count_ex(1, 0, rp.ctypes.data, None, tc.TC_SORTED, None,
                           ctypes.addressof(total), None, None) == EINVAL
    # bad shard arguments
    assert lib.tc_count_shard(1, 0, rp.ctypes.data, None, 0, None, 2, 2, rp.ctypes.data, None,
                              None) == EINVAL
    assert lib.tc_count_shard(1, 0, rp.ctypes.data, None, tc.TC_HOST_PTRS, None, 0, 2,
                              rp.ctypes.data, None, None) == EINVAL
    # bad forced variant / reserved bits
    o = tc.Options()
    lib.tc_default_options(ctypes.byref(o))
    o.force_variant = 7
    assert lib.tc_count_ex(1, 0, rp.ctypes.data, None, 0, ctypes.byref(o),
                           ctypes.addressof(total), None, None) == EINVAL
    lib.tc_default_options(ctypes.byref(o))
    o.reserved[3] = 1
    assert lib.tc_count_ex(1, 0, rp.ctypes.data, None, 0, ctypes.byref(o),
                           ctypes.addressof(total), None, None) == EINVAL
    # the workspace hook comes as a pair
    lib.tc_default_options(ctypes.byref(o))
    o.alloc = tc.ALLOC_FN(lambda c, size, stream: None)
    assert lib.tc_count_ex(1, 0, rp.ctypes.data, None, 0, ctypes.byref(o),
                           ctypes.addressof(total), None, None) == EINVAL
    assert b"together" in lib.tc_last_error()
    # tc_count reports failure as TC_ERROR
    assert lib.tc_count(1 << 32, 0, rp.ctypes.data, None, 0) == tc.TC_ERROR


def test_product_package_does_not_touch_oracle():
    """The product path never imports or links the oracle (independence)."""
    pkg = os.path.join(ROOT, "paper_1804_06926_b200")
    pat = re.compile(r"^\s*(import oracle|from oracle)|oracle_[a-z]+\(|liboracle", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f
    data = open(tc.library_path(), "rb").read()
    assert b"oracle_" not in data


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(tc, "_lib", None)
    monkeypatch.setattr(tc, "_LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        tc._load()
