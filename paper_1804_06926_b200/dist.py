"""Multi-GPU driver: one process per GPU, torch.distributed (NCCL).

Every rank holds the same input graph (replicated: an R-MAT s26 oriented CSR is
~5 GB, far below 180 GB of HBM), runs the identical preprocessing, and
``tc_count_shard`` keeps only the sources of its work-prefix group (no
communication for the split).  The single exchange step is ONE allreduce of
the int64 partial count (non-negative sums < 2^63, so two's-complement int64
addition equals uint64 addition bit for bit), plus an n-entry allreduce in
per-vertex mode.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import clean_shard, count_edges_shard, count_shard


class Comm:
    """The collectives of the sharded pipeline (shard.py) over a torch.distributed group:
    NCCL on GPUs (gloo on CPU tensors for the host-logic tests)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        # gloo (CPU tests; two ranks sharing one GPU in the GPU tests) stages CUDA tensors
        # through host memory; NCCL works on them directly
        self.stage = dist.get_backend(group) == "gloo"

    def _src(self, q):
        return dist.get_global_rank(self.group, q) if self.group is not None else q

    def all_reduce(self, t):
        if self.stage and t.is_cuda:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            t.copy_(h)
            return
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def all_to_all(self, send, counts, width):
        """send holds `width` elements per item, grouped by destination (counts[q] items for
        rank q); returns the items every rank sent here, grouped by source rank."""
        dev = send.device
        cdev = torch.device("cpu") if self.stage else dev
        sc = torch.tensor(counts, dtype=torch.int64, device=cdev)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        rcount = [int(x) for x in rc.tolist()]
        recv = torch.empty(width * sum(rcount), dtype=send.dtype, device=cdev)
        dist.all_to_all_single(recv, send[:width * sum(counts)].to(cdev),
                               output_split_sizes=[width * c for c in rcount],
                               input_split_sizes=[width * c for c in counts], group=self.group)
        return recv.to(dev)

    def broadcast_slices(self, buf, bounds, async_op=False):
        """All-gather of contiguous slices: rank q owns buf[bounds[q]:bounds[q+1]] (in place).
        async_op: NCCL broadcasts left in flight, returned for wait()."""
        works = []
        for q in range(self.world):
            if bounds[q + 1] > bounds[q]:
                sl = buf[bounds[q]:bounds[q + 1]]
                if self.stage and sl.is_cuda:
                    h = sl.cpu()
                    dist.broadcast(h, src=self._src(q), group=self.group)
                    sl.copy_(h)
                else:
                    w = dist.broadcast(sl, src=self._src(q), group=self.group, async_op=async_op)
                    if async_op:
                        works.append(w)
        return works

    def wait(self, works):
        for w in works or []:
            w.wait()


def count_distributed_sharded(rowptr: torch.Tensor, col: torch.Tensor, group=None, *,
                              per_vertex: bool = False, **opts):
    """Exact triangle count with a1-a5 sharded too (shard.py run_rank: six phases between the
    collectives of Comm) and one all-reduce of the partial count [and per-vertex partials]."""
    from .shard import run_rank
    comm = Comm(group)
    partial, pv = run_rank(rowptr, col, comm.rank, comm.world, comm, per_vertex=per_vertex, **opts)
    if per_vertex:
        both = torch.cat([partial, pv])
        comm.all_reduce(both)
        return int(both[0].item()), both[1:]
    comm.all_reduce(partial)
    return int(partial.item())


def exchange_clean_shards(rowptr: torch.Tensor, col: torch.Tensor, group=None, *, clean_fn=None):
    """Sharded a1 (tc_clean_shard on every rank) + its exchange: ONE all-reduce of the n int32
    degree partials and ONE all-gather of the ranks' cleaned edge lists (padded to the longest,
    the valid prefixes concatenated).  Returns (edges of every rank, summed degrees)."""
    world = dist.get_world_size(group)
    fn = clean_fn or clean_shard
    edges, deg = fn(rowptr, col, dist.get_rank(group), world)
    dist.all_reduce(deg, op=dist.ReduceOp.SUM, group=group)
    dev = deg.device
    m = torch.tensor([edges.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(m) for _ in range(world)]
    dist.all_gather(sizes, m, group=group)
    sizes = [int(x.item()) for x in sizes]
    pad = max(sizes) if sizes else 0
    buf = torch.zeros(pad, dtype=torch.int64, device=dev)
    buf[:edges.numel()] = edges
    out = [torch.empty(pad, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([o[:s] for o, s in zip(out, sizes)]), deg


def count_distributed_sharded_a1(rowptr: torch.Tensor, col: torch.Tensor, group=None, *,
                                 per_vertex: bool = False, clean_fn=None, count_fn=None):
    """count_distributed with the cleaning step (a1) split over the ranks instead of repeated:
    exchange_clean_shards, then tc_count_edges_shard on the gathered edges and one all-reduce
    of the partial count (and of the per-vertex partials)."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n = rowptr.numel() - 1
    edges, deg = exchange_clean_shards(rowptr, col, group, clean_fn=clean_fn)
    dev = rowptr.device
    partial = torch.zeros(1, dtype=torch.int64, device=dev)
    pv = torch.zeros(n, dtype=torch.int64, device=dev) if per_vertex else None
    (count_fn or count_edges_shard)(n, edges, deg, rank, world, partial, per_vertex_partial=pv)
    if per_vertex:
        both = torch.cat([partial, pv])
        dist.all_reduce(both, op=dist.ReduceOp.SUM, group=group)
        return int(both[0].item()), both[1:]
    dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return int(partial.item())


def count_distributed(rowptr: torch.Tensor, col: torch.Tensor, group=None, *, shard_fn=None,
                      per_vertex: bool = False, **kw):
    """Exact triangle count of the replicated graph, summed over the ranks of `group`.

    `shard_fn(rowptr, col, rank, world, partial, per_vertex_partial=..., **kw)` defaults to the
    CUDA library's tc_count_shard; tests on CPU (gloo) inject a stand-in.
    """
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    fn = shard_fn or count_shard
    dev = rowptr.device
    partial = torch.zeros(1, dtype=torch.int64, device=dev)
    pv = torch.zeros(rowptr.numel() - 1, dtype=torch.int64, device=dev) if per_vertex else None
    fn(rowptr, col, rank, world, partial, per_vertex_partial=pv, **kw)
    if per_vertex:
        both = torch.cat([partial, pv])
        dist.all_reduce(both, op=dist.ReduceOp.SUM, group=group)
        return int(both[0].item()), both[1:]
    dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
    return int(partial.item())
