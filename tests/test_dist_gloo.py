"""World-size-2 CPU (gloo) test of the multi-GPU driver's host logic (dist.py):
process-group plumbing, the int64 allreduce of partial counts, and the per-vertex
allreduce.  The per-rank shard here is a CPU stand-in -- the oracle counting one
connected component of a disjoint union per rank -- because no GPU is present; the CUDA
partition itself is covered by tests/test_gpu_parity.py::test_shards_sum_to_total."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _parts():
    import graphgen as G
    return [G.karate(), G.rmat(9, 16, seed=3)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import graphgen as G
        import oracle as O
        from paper_1804_06926_b200.dist import count_distributed

        parts = _parts()
        g = G.disjoint_union(*parts)
        offsets = np.cumsum([0] + [p.n for p in parts])

        def shard_fn(rowptr, col, r, w, partial, per_vertex_partial=None, **kw):
            assert (r, w) == (rank, world)
            p = parts[r]
            T, t = O.count(p.n, p.rowptr, p.col, per_vertex=True)
            partial.fill_(T)
            if per_vertex_partial is not None:
                per_vertex_partial.zero_()
                per_vertex_partial[offsets[r]:offsets[r + 1]] = torch.from_numpy(t.astype(np.int64))

        rp = torch.from_numpy(g.rowptr.view(np.int64))
        cl = torch.from_numpy(g.col.view(np.int32))
        T = count_distributed(rp, cl, shard_fn=shard_fn)
        T2, pv = count_distributed(rp, cl, shard_fn=shard_fn, per_vertex=True)
        q.put((rank, T, T2, pv.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_allreduce_wiring_world2():
    import graphgen as G
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = G.disjoint_union(*_parts())
    T, t = O.count(g.n, g.rowptr, g.col, per_vertex=True)
    for rank, T1, T2, pv in res:
        assert T1 == T and T2 == T
        assert (pv.astype(np.uint64) == t).all()


def _clean_worker(rank, world, port, q):
    """exchange_clean_shards' wiring (degree all-reduce, variable-size edge all-gather) with a
    CPU stand-in for tc_clean_shard: this rank's edges = the clean edges whose smaller endpoint
    is = rank (mod world), as (min << b) | max keys, and the degrees they contribute."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import graphgen as G
        import oracle as O
        from paper_1804_06926_b200.dist import exchange_clean_shards

        g = G.dirty(G.gnp(400, 0.05, 2), seed=3)
        b = max(1, (g.n - 1).bit_length())

        def clean_fn(rowptr, col, r, w):
            crow, ccol = O.clean(g.n, g.rowptr, g.col)
            src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(crow).astype(np.int64))
            dst = ccol.astype(np.int64)
            keep = (src < dst) & (src % w == r)
            keys = (src[keep] << b) | dst[keep]
            deg = np.bincount(src[keep], minlength=g.n) + np.bincount(dst[keep], minlength=g.n)
            return torch.from_numpy(keys), torch.from_numpy(deg.astype(np.int32))

        rp = torch.from_numpy(g.rowptr.view(np.int64))
        cl = torch.from_numpy(g.col.view(np.int32))
        edges, deg = exchange_clean_shards(rp, cl, clean_fn=clean_fn)
        q.put((rank, np.sort(edges.numpy()), deg.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_clean_shard_exchange_world2():
    import graphgen as G
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_clean_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = G.dirty(G.gnp(400, 0.05, 2), seed=3)
    crow, ccol = O.clean(g.n, g.rowptr, g.col)
    b = max(1, (g.n - 1).bit_length())
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(crow).astype(np.int64))
    dst = ccol.astype(np.int64)
    want = np.sort(((src << b) | dst)[src < dst])
    for rank, keys, deg in res:
        assert (keys == want).all(), rank
        assert (deg == np.diff(crow)).all(), rank


# ------------------------------------------------------------------ sharded pipeline collectives
def _comm_worker(rank, world, port, q):
    """dist.Comm (the sharded pipeline's collectives, shard.py run_rank) under gloo: all-to-all
    of width-3 items with uneven counts, slice all-gather by broadcasts, all-reduce."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1804_06926_b200.dist import Comm
        comm = Comm()
        counts = [rank + 1 + 2 * d for d in range(world)]          # items for destination d
        send = torch.cat([torch.arange(3 * c, dtype=torch.int32) + 1000 * rank + 100 * d
                          for d, c in enumerate(counts)])
        recv = comm.all_to_all(send, counts, 3)
        bounds = [0, 3, 10][:world + 1]
        buf = torch.full((bounds[world],), -1, dtype=torch.int32)
        buf[bounds[rank]:bounds[rank + 1]] = rank + 7
        comm.broadcast_slices(buf, bounds)
        t = torch.tensor([rank + 1, 10 * rank], dtype=torch.int64)
        comm.all_reduce(t)
        q.put((rank, recv.numpy().copy(), buf.numpy().copy(), t.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_sharded_comm_world2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, recv, buf, t = q.get(timeout=120)
        res[r] = (recv, buf, t)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        # what shard.emulate builds locally: every source's chunk for r, in source order
        want = np.concatenate([np.arange(3 * (s + 1 + 2 * r), dtype=np.int32) + 1000 * s + 100 * r
                               for s in range(world)])
        assert (res[r][0] == want).all()
        assert (res[r][1] == np.array([7, 7, 7] + [8] * 7, np.int32)).all()
        assert (res[r][2] == np.array([3, 10])).all()
