"""Multi-GPU plans for the DBSA hot path.

Three strategies, one process per GPU:

* **Stage 2, query data-parallel.**  Test queries are independent
  (`Runner.infer` is pure given weights, cache and index; pipeline.py:322-327).
  Each rank answers its slice of the queries (`query_slice`), and the
  predictions are gathered at the end (`gather_predictions`).
* **Stage 1, group-sharded with a per-layer halo.**  With sink-prev-self(j),
  group i at layer l needs groups i-1 .. i-j at layer l (masks.py:91-97), so
  ranks own contiguous group ranges (`plan_group_shards`).  Each rank encodes
  the sink group 0 redundantly: `context_ids(0) = ()`, so no sink traffic.
  Per layer, every rank sends the K/V pages of the groups its successors
  need (`halo_plan`, `exchange_pages`).  This is about 12 MB per layer at
  C2 (two 1,500-token groups × 8 kv heads × 128 × K/V × bf16).
* **Group-sharded cache (C5).**  Pages stay on the rank that encoded them.
  A query's chunk table is split by owner.  Each rank computes an
  (O partial, LSE) for every query row over its local chunks; exactly one
  rank, the "self rank", also covers the query's own tokens.  The partials
  are all-gathered per layer and merged by K3m (`dbsa_lse_merge` with
  split_stride = rows per rank).

`Comm` hides the transport.
* `DistComm` wraps torch.distributed (NCCL on GPUs, gloo for the CPU tests).
* `LocalComm` runs N logical shards inside one process. This is the
  single-GPU "logical shard" mode SURVEY.md §4 recommends for testing the
  sharded algorithms against the unsharded result.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


# ------------------------------------------------------------------ plans
def query_slice(n_queries: int, world: int, rank: int) -> slice:
    """Contiguous ceil-split of the query list (stage-2 query DP)."""
    per = -(-n_queries // world)
    return slice(min(n_queries, rank * per), min(n_queries, (rank + 1) * per))


def plan_group_shards(counts, world: int) -> list[tuple[int, int]]:
    """Contiguous [g0, g1) ranges of groups 1..B-1 balanced by token count.

    Group 0 (the sink) belongs to rank 0 and is re-encoded by every rank.
    A rank may own an empty range when there are fewer groups than ranks.
    """
    counts = np.asarray(counts, dtype=np.int64)
    b = len(counts)
    if world < 1:
        raise ValueError("world must be >= 1")
    cum = np.cumsum(counts[1:]) if b > 1 else np.zeros(0, np.int64)
    total = int(cum[-1]) if len(cum) else 0
    bounds = [1]
    for r in range(1, world):
        k = int(np.searchsorted(cum, total * r / world, side="left")) + 1
        bounds.append(min(max(k, bounds[-1]), b))
    bounds.append(b)
    ranges = [(bounds[r], bounds[r + 1]) for r in range(world)]
    g0, g1 = ranges[0]
    ranges[0] = (0, g1)
    return ranges


def owner_of(group: int, ranges) -> int:
    for r, (a, b) in enumerate(ranges):
        if a <= group < b:
            return r
    raise KeyError(f"group {group} owned by no rank")


def local_groups(pattern, ranges, rank: int, n_blocks: int) -> list[int]:
    """Groups whose pages rank `rank` holds during stage 1: its own range, the
    sink, and the context groups of its own groups (the halo)."""
    a, b = ranges[rank]
    need = set(range(a, b)) | {0}
    for g in range(a, b):
        need |= set(pattern.context_of(g))
    return sorted(x for x in need if x < n_blocks)


def halo_plan(pattern, ranges, n_blocks: int) -> list[tuple[int, int, int]]:
    """(group, src rank, dst rank) for every context group a rank needs but does
    not own; the sink is excluded (every rank computes it)."""
    out = []
    for dst in range(len(ranges)):
        for g in local_groups(pattern, ranges, dst, n_blocks):
            if g == 0:
                continue
            src = owner_of(g, ranges)
            if src != dst:
                out.append((g, src, dst))
    return out


def split_chunks_by_owner(units, ranges) -> dict[int, list[int]]:
    """Indices of a query's ordered units per owner rank (C5 stage 2).  Units
    keep their global new positions, so the RoPE shift stays correct."""
    out: dict[int, list[int]] = {}
    for i, u in enumerate(units):
        out.setdefault(owner_of(u.block_id if hasattr(u, "block_id") else int(u[0]), ranges), []).append(i)
    return out


def merge_partials_reference(part_o, part_lse):
    """Test oracle of the K3m merge over a leading split axis (torch, any
    device): lse = logsumexp_s lse_s, O = sum_s exp(lse_s - lse) O_s."""
    import torch

    lse = torch.logsumexp(part_lse, dim=0)
    w = torch.exp(part_lse - lse.unsqueeze(0))
    w = torch.nan_to_num(w, nan=0.0)
    return (w.unsqueeze(-1) * part_o).sum(0), lse


# ------------------------------------------------------------------ transports
class LocalComm:
    """N logical shards in one process: collectives are list operations."""

    def __init__(self, n: int):
        self.world = n
        self.local_ranks = list(range(n))

    def exchange(self, sends):
        """sends: {(src, dst, key): tensor}; returns {(src, dst, key): tensor} as
        received on dst (the same tensors: shards share the device)."""
        return dict(sends)

    def all_gather(self, parts):
        """parts: [tensor per local rank] -> stacked [world, ...]."""
        import torch

        return torch.stack(parts, 0)

    def all_gather_object(self, obj_per_rank):
        return list(obj_per_rank)


class DistComm:
    """torch.distributed transport: one local rank per process.  NCCL moves
    device tensors directly over NVLink; under gloo (the CPU tests, and the
    two-process test of the sharded paths on ONE GPU, where NCCL cannot run
    two ranks on one device) device tensors are staged through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.local_ranks = [self.rank]
        self.host_staged = dist.get_backend(group) == "gloo"
        # a collective every rank joins, before any batched P2P (NCCL requirement)
        dist.barrier(group=group)

    def exchange(self, sends, recv_like=None):
        """Point-to-point halo exchange.  sends: {(src, dst, key): tensor} for
        src == this rank; recv_like: {(src, dst, key): empty tensor} for dst ==
        this rank.  Returns the received tensors."""
        ops = []
        for (src, dst, key), t in sorted(sends.items()):
            t = t.contiguous()
            ops.append(self.dist.P2POp(self.dist.isend, t.cpu() if self.host_staged else t, dst, self.group))
        out, staged = {}, []
        for (src, dst, key), t in sorted((recv_like or {}).items()):
            out[(src, dst, key)] = t
            buf = t.cpu() if self.host_staged and t.is_cuda else t
            if buf is not t:
                staged.append((buf, t))
            ops.append(self.dist.P2POp(self.dist.irecv, buf, src, self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        for buf, t in staged:
            t.copy_(buf)
        return out

    def all_gather(self, parts):
        import torch

        (part,) = parts
        part = part.contiguous()
        if self.host_staged:
            bufs = [torch.empty(part.shape, dtype=part.dtype) for _ in range(self.world)]
            self.dist.all_gather(bufs, part.cpu(), group=self.group)
            return torch.stack(bufs, 0).to(part.device)
        out = torch.empty((self.world * part.shape[0],) + tuple(part.shape[1:]), dtype=part.dtype,
                          device=part.device)
        self.dist.all_gather_into_tensor(out, part, group=self.group)
        return out.view((self.world,) + tuple(part.shape))

    def all_gather_object(self, obj_per_rank):
        (obj,) = obj_per_rank
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


def gather_predictions(comm, local_preds):
    """Concatenate per-rank prediction lists in rank order (stage-2 query DP)."""
    lists = comm.all_gather_object([list(local_preds)])
    return [p for part in lists for p in part]


# ------------------------------------------------------------------ page slices
@dataclass(frozen=True)
class PageSlice:
    """The rows of one group in one layer of a page store."""

    layer: int
    row0: int
    n_rows: int


def pack_pages(k_planes, v_planes, sl: PageSlice):
    """Copy one group's K rows and V^T columns of one layer into one contiguous
    buffer: [Hkv, n_rows, HDP] K followed by [Hkv, HDP, n_rows] V^T."""
    import torch

    k = k_planes[sl.layer, :, sl.row0:sl.row0 + sl.n_rows, :]
    v = v_planes[sl.layer, :, :, sl.row0:sl.row0 + sl.n_rows]
    return torch.cat([k.reshape(-1), v.reshape(-1)])


def unpack_pages(buf, k_planes, v_planes, sl: PageSlice):
    hkv, hdp = k_planes.shape[1], k_planes.shape[3]
    nk = hkv * sl.n_rows * hdp
    k_planes[sl.layer, :, sl.row0:sl.row0 + sl.n_rows, :].copy_(buf[:nk].view(hkv, sl.n_rows, hdp))
    v_planes[sl.layer, :, :, sl.row0:sl.row0 + sl.n_rows].copy_(buf[nk:].view(hkv, hdp, sl.n_rows))


def exchange_pages(comm, layer: int, plan, stores, entries):
    """Per-layer halo exchange of stage 1.

    plan: (group, src, dst) triples (halo_plan).  stores: {rank: PageStore}
    for the local ranks.  entries: {rank: {group: BlockEntry}} giving each
    local rank's row of each group it holds.  Sends the group's rows of
    `layer` from src's store into dst's store.
    """
    import torch

    local = set(comm.local_ranks)
    sends, recv_like, targets = {}, {}, []
    for g, src, dst in plan:
        if src in local:
            e = entries[src][g]
            n_rows = -(-e.token_count // 64) * 64
            sends[(src, dst, g)] = pack_pages(stores[src].k, stores[src].v, PageSlice(layer, e.row0, n_rows))
        if dst in local:
            e = entries[dst][g]
            n_rows = -(-e.token_count // 64) * 64
            st = stores[dst]
            numel = st.k.shape[1] * n_rows * st.k.shape[3] * 2
            if src not in local:
                recv_like[(src, dst, g)] = torch.empty(numel, dtype=st.k.dtype, device=st.k.device)
            targets.append(((src, dst, g), st, PageSlice(layer, e.row0, n_rows)))
    if isinstance(comm, LocalComm):
        received = sends
    else:
        received = comm.exchange({k: v for k, v in sends.items() if k[1] not in local}, recv_like)
        received.update({k: v for k, v in sends.items() if k[1] in local})
    for key, st, sl in targets:
        unpack_pages(received[key], st.k, st.v, sl)
