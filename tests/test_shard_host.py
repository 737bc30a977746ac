"""CPU test of the sharded pipeline's host logic (shard.emulate, the one-GPU stand-in of the
collectives dist.Comm runs with NCCL): the six phase calls are replaced by stand-ins that tag
every item with (source rank, destination rank, index), so the test checks what the emulation
hands each rank -- the summed degree / d+ / owner-work arrays, every rank's pairs and entries
routed to their destination in source-rank order, one col+ buffer written slice by slice --
and that the partial counts are summed.  (tests/test_dist_gloo.py checks that dist.Comm's
collectives produce exactly these local concatenations; tests/test_gpu_shard.py runs the real
phases against the oracle.)"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1804_06926_b200 import shard  # noqa: E402

N, WORLD = 40, 3


def _tag(src, dst, k):
    return src * 1_000_000 + dst * 1_000 + k


@pytest.fixture
def fake_phases(monkeypatch):
    seen = {"rows": {}, "count": {}}

    def clean_shard(rowptr, col, r, world, **kw):
        deg = torch.full((N,), r + 1, dtype=torch.int32)
        return torch.arange(5, dtype=torch.int64) + 100 * r, deg

    def shard_orient(n, edges, deg, **kw):
        r = int(edges[0]) // 100
        assert (deg == sum(range(1, WORLD + 1))).all()            # degrees all-reduced
        newid = torch.arange(n, dtype=torch.int32)
        dplus = torch.full((n,), 10 * (r + 1), dtype=torch.int32)
        src = torch.full((4,), r, dtype=torch.int32)
        return newid, src, src.clone(), dplus

    def shard_partition(n, src, dst, dplus, r, world, **kw):
        assert (dplus == sum(10 * (q + 1) for q in range(world))).all()   # d+ all-reduced
        counts = [q + 1 for q in range(world)]                    # q + 1 pairs for rank q
        pairs = torch.cat([torch.tensor([_tag(r, q, k) for k in range(c)], dtype=torch.int64)
                           for q, c in enumerate(counts)])
        rows = list(range(0, n + 1, n // world))[:world] + [n]
        cb = [0]
        for q in range(world):                                    # rank q's slice: q+1 items per source
            cb.append(cb[-1] + world * (q + 1))
        off = torch.zeros(n + 1, dtype=torch.int64)
        return off, pairs, counts, rows, cb

    def shard_rows(n, pairs, col_plus, col_begin, **kw):
        q = int(pairs[0]) // 1_000 % 1_000
        want = [_tag(s, q, k) for s in range(WORLD) for k in range(q + 1)]
        assert pairs.tolist() == want                             # every source's chunk, in order
        col_plus[col_begin:col_begin + len(pairs)] = q + 1
        seen["rows"][q] = col_begin

    def shard_work(n, off, col_plus, dplus, r0, r1, e0, e1, **kw):
        r = [q for q, b in seen["rows"].items() if b == e0][0]
        assert (col_plus[e0:e1] == r + 1).all()                   # its slice of the shared col+
        return (torch.full((n,), 1, dtype=torch.int32), torch.full((n,), 2, dtype=torch.int64),
                torch.full((n,), 3, dtype=torch.int32))

    def shard_route(n, off, col_plus, dplus, cnt, ln, spans, r, world, e0, e1, **kw):
        assert (cnt == world).all() and (ln == 2 * world).all() and (spans == 3 * world).all()
        counts = [2 * (q + 1) for q in range(world)]
        ent = torch.cat([torch.tensor([_tag(r, q, k) for k in range(3 * c)], dtype=torch.int32)
                         for q, c in enumerate(counts)])
        return ent, counts

    def shard_count(n, off, col_plus, dplus, newid, entries, r, world, e0, e1, partial, **kw):
        want = [_tag(s, r, k) for s in range(world) for k in range(3 * 2 * (r + 1))]
        assert entries.tolist() == want                           # entries routed to their owner
        partial.fill_(entries.numel() // 3)
        seen["count"][r] = True

    for name, fn in [("clean_shard", clean_shard), ("shard_orient", shard_orient),
                     ("shard_partition", shard_partition), ("shard_rows", shard_rows),
                     ("shard_work", shard_work), ("shard_route", shard_route),
                     ("shard_count", shard_count)]:
        monkeypatch.setattr(shard, name, fn)
    return seen


def test_emulate_routes_and_sums(fake_phases):
    rowptr = torch.zeros(N + 1, dtype=torch.int64)
    col = torch.zeros(1, dtype=torch.int32)
    total, pv, rep = shard.emulate(rowptr, col, WORLD)
    # rank r received 2(r+1) entries from each of the WORLD ranks
    assert total == sum(WORLD * 2 * (r + 1) for r in range(WORLD))
    assert pv is None
    assert sorted(fake_phases["rows"]) == list(range(WORLD))
    assert sorted(fake_phases["count"]) == list(range(WORLD))
