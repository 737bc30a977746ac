"""bench.py's N > 1 code path end to end on the one GPU of this round's boxes: two ranks on
cuda:0 over gloo (TC_BENCH_SHARED_GPU=1; NCCL refuses two ranks on one device), launched the
way the driver launches it (bench.py --gpus 2 re-spawns itself under torch.distributed.run).
The line must carry n_gpus 2 and the oracle's T for every multi-GPU mode (the timings of two
ranks sharing a GPU mean nothing)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode", [[], ["--sharded-a1-only"], ["--replicated-a1"]])
def test_bench_two_ranks(mode):
    import graphgen as G
    import oracle as O
    g = G.rmat(14, 16)
    T = O.count(g.n, g.rowptr, g.col)
    env = dict(os.environ, TC_BENCH_SHARED_GPU="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
                        "--warmup", "3", "--scale", "14", *mode], capture_output=True, text=True,
                       timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = lines[0]
    assert line["n_gpus"] == 2 and line["config"]["T"] == T
    assert line["gpu_launches"] > 0 and line["e2e"]["value"] > 0


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("mode", [[], ["--sharded-a1-only"], ["--replicated-a1"]])
def test_bench_nccl_one_rank(mode):
    """The N > 1 path over REAL NCCL (dist.Comm without host staging: all_to_all_single with
    splits, async broadcasts, all-reduces on CUDA tensors), one rank under torch.distributed.run
    (TC_BENCH_FORCE_DIST=1): the 1-GPU box cannot host two NCCL ranks, but every collective
    call, dtype and stream hand-off of the multi-GPU job runs."""
    import graphgen as G
    import oracle as O
    g = G.rmat(14, 16)
    T = O.count(g.n, g.rowptr, g.col)
    env = dict(os.environ, TC_BENCH_FORCE_DIST="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                        "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
                        os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "2", "--warmup", "3",
                        "--scale", "14", *mode], capture_output=True, text=True, timeout=600, env=env,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = lines[0]
    assert line["config"]["T"] == T and line["gpu_launches"] > 0 and line["e2e"]["value"] > 0
