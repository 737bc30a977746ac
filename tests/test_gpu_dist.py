"""The multi-GPU paths end to end through the REAL library (the gloo test used an
oracle stand-in shard): world-2 process group, both ranks on cuda:0 (the round's boxes have
one GPU; NCCL refuses two ranks on one device, so the group is gloo over CUDA tensors), each
rank running paper_1804_06926_b200.dist.count_distributed -> tc_count_shard + allreduce.
The sums must equal the oracle bit for bit (total and every t(v))."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _graph(name):
    import graphgen as G
    return {"rmat15": lambda: G.rmat(15, 16, seed=8), "clique": lambda: G.clique_union(20_000, 30_000)}[name]()


def _worker(rank, world, port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1804_06926_b200.dist import (count_distributed, count_distributed_sharded,
                                                count_distributed_sharded_a1)
        g = _graph(name)
        dev = torch.device("cuda:0")
        rp = torch.from_numpy(g.rowptr.view(np.int64)).to(dev)
        cl = torch.from_numpy(g.col.view(np.int32)).to(dev)
        T = count_distributed(rp, cl)
        T2, pv = count_distributed(rp, cl, per_vertex=True)
        # the cleaning step split over the ranks: one degree all-reduce + one edge all-gather
        T3 = count_distributed_sharded_a1(rp, cl)
        T4, pv4 = count_distributed_sharded_a1(rp, cl, per_vertex=True)
        assert T3 == T and T4 == T and (pv4 == pv).all()
        # a1-a5 sharded (shard.py run_rank through dist.Comm: all-reduce, all-to-all, broadcasts)
        T5 = count_distributed_sharded(rp, cl)
        T6, pv6 = count_distributed_sharded(rp, cl, per_vertex=True)
        assert T5 == T and T6 == T and (pv6 == pv).all()
        q.put((rank, T, T2, pv.cpu().numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["rmat15", "clique"])
def test_count_distributed_world2_real_shards(name):
    import oracle as O
    g = _graph(name)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, T1, T2, pv in res:
        assert T1 == T and T2 == T, rank
        assert (pv.astype(np.uint64) == t).all(), rank


def _nccl_worker(port, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        from paper_1804_06926_b200.dist import (count_distributed, count_distributed_sharded,
                                                count_distributed_sharded_a1)
        g = _graph(name)
        dev = torch.device("cuda:0")
        rp = torch.from_numpy(g.rowptr.view(np.int64)).to(dev)
        cl = torch.from_numpy(g.col.view(np.int32)).to(dev)
        out = [count_distributed(rp, cl), count_distributed_sharded_a1(rp, cl),
               count_distributed_sharded(rp, cl)]
        T, pv = count_distributed_sharded(rp, cl, per_vertex=True)
        q.put((out + [T], pv.cpu().numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["rmat15", "clique"])
def test_count_distributed_nccl_world1(name):
    """The three distributed drivers over a REAL NCCL group (one rank on the one GPU): the NCCL
    collectives of dist.Comm run on CUDA tensors (no host staging)."""
    import oracle as O
    g = _graph(name)
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), name, q))
    p.start()
    got, pv = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert got == [T] * 4
    assert (pv.astype(np.uint64) == t).all()
