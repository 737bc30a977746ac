"""tc_options.graph_cache (tc_api.cu): the count captured into a CUDA graph on first use and
replayed by later calls with the same arguments.  Every replay must equal the oracle -- also
after the input buffers are rewritten in place with ANOTHER graph of the same n and m (the
graph holds no data-dependent host decision: every size it was built with is n, m or a
device-side count), with per-vertex output, on clean input, and next to non-graph calls."""
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


@pytest.mark.parametrize("scale", [10, 14])
def test_graph_replay_matches_oracle(scale):
    g1 = G.rmat(scale, 16, seed=1)
    g2 = G.rmat(scale, 16, seed=2)          # same n and m (R-MAT: n = 2^s, m = 16 n raw arcs)
    assert g1.n == g2.n and g1.arcs == g2.arcs
    T1, t1 = O.count(g1.n, g1.rowptr, g1.col, per_vertex=True)
    T2, t2 = O.count(g2.n, g2.rowptr, g2.col, per_vertex=True)
    rp, cl = on_dev(g1.rowptr, g1.col)
    pv = torch.zeros(g1.n, dtype=torch.int64, device=DEV)
    for _ in range(3):   # capture, then replays
        assert tc.count_ex(rp, cl, graph_cache=1, tiny_max_n=0, lowdeg_max=0) == T1
    l0 = tc.launches_issued()
    assert tc.count_ex(rp, cl, graph_cache=1, tiny_max_n=0, lowdeg_max=0) == T1
    assert tc.launches_issued() - l0 > 10          # the replayed graph's kernels are counted
    # same buffers, new content: the replay recomputes everything
    r2, c2 = on_dev(g2.rowptr, g2.col)
    rp.copy_(r2)
    cl.copy_(c2)
    torch.cuda.synchronize()
    assert tc.count_ex(rp, cl, graph_cache=1, tiny_max_n=0, lowdeg_max=0) == T2
    assert tc.count_ex(rp, cl, tiny_max_n=0, lowdeg_max=0) == T2                 # and without the graph
    got, pvo = tc.count_ex(rp, cl, per_vertex=True, graph_cache=1, tiny_max_n=0, lowdeg_max=0)
    got, pvo = tc.count_ex(rp, cl, per_vertex=True, graph_cache=1, tiny_max_n=0, lowdeg_max=0)
    torch.cuda.synchronize()
    assert got == T2 and (pvo.cpu().numpy().view(np.uint64) == t2).all()


def test_graph_replay_clean_input_and_tiny():
    g = G.rmat(12, 16, seed=7)
    T = O.count(g.n, g.rowptr, g.col)
    row, col = O.clean(g.n, g.rowptr, g.col)
    rp, cl = on_dev(row, col)
    for _ in range(3):
        assert tc.count_ex(rp, cl, clean=True, sorted_rows=True, graph_cache=1) == T
    k = G.karate()
    kr, kc = on_dev(k.rowptr, k.col)
    for _ in range(3):   # the one-kernel path captured too
        assert tc.count_ex(kr, kc, graph_cache=1) == 45


def test_trim_drops_replay_graphs():
    g = G.rmat(11, 16, seed=3)
    T = O.count(g.n, g.rowptr, g.col)
    rp, cl = on_dev(g.rowptr, g.col)
    for _ in range(2):
        assert tc.count_ex(rp, cl, graph_cache=1, tiny_max_n=0, lowdeg_max=0) == T
    tc.trim_workspace()
    for _ in range(2):   # captured again after the trim
        assert tc.count_ex(rp, cl, graph_cache=1, tiny_max_n=0, lowdeg_max=0) == T
