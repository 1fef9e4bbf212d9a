"""Multi-process (gloo, world size 2) and plan tests of the multi-GPU layer
(paper_2503_08640_b200/parallel.py), on CPU.  The GPU kernels are not
involved: these cover group sharding, the stage-1 halo plan and its page
exchange, the stage-2 query split / prediction gather, and the algebra of
the C5 LSE merge.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_08640_b200 import masks, parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_group_shards_cover_and_balance():
    counts = [40] + [1500] * 59
    for world in (1, 2, 3, 4, 8):
        r = parallel.plan_group_shards(counts, world)
        assert r[0][0] == 0 and r[-1][1] == 60
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        sizes = [sum(counts[max(a, 1):b]) for a, b in r]
        assert max(sizes) - min(sizes) <= 1500
    # more ranks than groups: empty ranges, still a cover
    r = parallel.plan_group_shards([10, 10, 10], 5)
    assert r[0][0] == 0 and r[-1][1] == 3 and sum(b - a for a, b in r) == 3


def test_halo_plan_sink_prev_self():
    pat = masks.AttentionPattern.sink_prev_self(2)
    ranges = [(0, 20), (20, 40), (40, 60)]
    plan = parallel.halo_plan(pat, ranges, 60)
    # rank 1 needs groups 18, 19 from rank 0; rank 2 needs 38, 39 from rank 1; the sink is never sent
    assert sorted(plan) == [(18, 0, 1), (19, 0, 1), (38, 1, 2), (39, 1, 2)]
    assert parallel.local_groups(pat, ranges, 1, 60) == [0, 18, 19] + list(range(20, 40))
    # self / sink-self patterns are embarrassingly parallel
    assert parallel.halo_plan(masks.AttentionPattern.sink_self(), ranges, 60) == []
    # a narrow range whose predecessors span two ranks
    plan = parallel.halo_plan(pat, [(0, 3), (3, 4), (4, 8)], 8)
    assert (2, 0, 2) in plan and (3, 1, 2) in plan and (1, 0, 1) in plan and (2, 0, 1) in plan


def test_query_slice_partition():
    for n in (0, 1, 7, 64, 4096):
        for world in (1, 2, 3, 8):
            idx = [i for r in range(world) for i in range(n)[parallel.query_slice(n, world, r)]]
            assert idx == list(range(n))


def test_lse_merge_reference_equals_single_softmax():
    g = torch.Generator().manual_seed(0)
    q = torch.randn(5, 16, generator=g, dtype=torch.float64)
    k = torch.randn(40, 16, generator=g, dtype=torch.float64)
    v = torch.randn(40, 16, generator=g, dtype=torch.float64)
    s = q @ k.T
    full = torch.softmax(s, -1) @ v
    cuts = [(0, 13), (13, 13), (13, 40)]  # includes an empty shard (LSE = -inf)
    po, pl = [], []
    for a, b in cuts:
        if b > a:
            ss = s[:, a:b]
            lse = torch.logsumexp(ss, -1)
            po.append(torch.softmax(ss, -1) @ v[a:b])
            pl.append(lse)
        else:
            po.append(torch.zeros(5, 16, dtype=torch.float64))
            pl.append(torch.full((5,), -float("inf"), dtype=torch.float64))
    o, lse = parallel.merge_partials_reference(torch.stack(po), torch.stack(pl))
    assert torch.allclose(o, full, atol=1e-12)
    assert torch.allclose(lse, torch.logsumexp(s, -1), atol=1e-12)


class _Store:
    def __init__(self, rows, hkv=2, hdp=16, layers=3, fill=0.0):
        self.k = torch.full((layers, hkv, rows, hdp), fill, dtype=torch.bfloat16)
        self.v = torch.full((layers, hkv, hdp, rows), fill, dtype=torch.bfloat16)


class _Entry:
    def __init__(self, row0, n):
        self.row0, self.token_count = row0, n


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = parallel.DistComm()
        pat = masks.AttentionPattern.sink_prev_self(2)
        counts = [70, 64, 100, 64, 30]
        ranges = parallel.plan_group_shards(counts, world)
        plan = parallel.halo_plan(pat, ranges, len(counts))
        present = parallel.local_groups(pat, ranges, rank, len(counts))
        # page rows of the present groups, in ascending order
        rows, entries, r0 = {}, {}, 0
        for g in present:
            entries[g] = _Entry(r0, counts[g])
            r0 += -(-counts[g] // 64) * 64
        store = _Store(r0)
        owned = set(range(*ranges[rank])) | {0}
        gen = torch.Generator().manual_seed(1)
        truth = {}
        for g in range(len(counts)):  # the same "true" pages on every rank
            n = -(-counts[g] // 64) * 64
            truth[g] = (torch.randn(3, 2, n, 16, generator=gen).to(torch.bfloat16),
                        torch.randn(3, 2, 16, n, generator=gen).to(torch.bfloat16))
        for g in owned & set(present):
            e = entries[g]
            n = -(-counts[g] // 64) * 64
            store.k[:, :, e.row0:e.row0 + n] = truth[g][0]
            store.v[..., e.row0:e.row0 + n] = truth[g][1]
        for layer in range(3):
            parallel.exchange_pages(comm, layer, plan, {rank: store}, {rank: entries})
        ok = True
        for g in present:
            e = entries[g]
            n = -(-counts[g] // 64) * 64
            ok &= torch.equal(store.k[:, :, e.row0:e.row0 + n], truth[g][0])
            ok &= torch.equal(store.v[..., e.row0:e.row0 + n], truth[g][1])
        preds = parallel.gather_predictions(comm, [f"r{rank}q{i}" for i in range(rank + 1)])
        # C5 partial all-gather layout: [world, R, hd]
        part = torch.full((6, 4), float(rank))
        gathered = comm.all_gather([part])
        ok &= gathered.shape == (world, 6, 4) and all(torch.all(gathered[r] == r) for r in range(world))
        q.put((rank, bool(ok), preds, [tuple(p) for p in plan]))
    finally:
        dist.destroy_process_group()


def test_two_rank_halo_exchange_and_gathers_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, preds, plan in res:
        assert ok, f"rank {rank}: halo pages or all-gather mismatch"
        assert preds == ["r0q0", "r1q0", "r1q1"]
        assert plan  # the 2-rank split of 5 groups needs a halo
