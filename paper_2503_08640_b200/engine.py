"""Device orchestration of the DBSA hot path on one B200.

Stage 1 (reference: pipeline.encode_blocks, pipeline.py:166-233) runs
LAYER-SYNCHRONOUSLY over all new groups at once -- legal because splitting at
group boundaries equals one forward under the token-level mask
(test_model.py:152-170, test_acceptance.py:60-108): per layer one QKV GEMM
over every pool token, one K2w launch writing every group's rotated K and V^T
into its pages, one K1 launch in which every CTA streams [sink, prev-j groups,
self-causal] for a 256-row slab of one group, then O-proj and FFN.

Stage 2 (reference: Runner.infer / score_label, pipeline.py:369-421,
model.py:420-443) scores ALL labels of a query in one forward: the query
tokens followed by every label, each label at positions T'+|q|.., with a tree
mask (label tokens see the query and their own label, causally) -- so the
selected KV is read once per query, not once per label.  Queries are batched:
the dense GEMMs see every new token of the batch, and K3 runs one CTA per
(query, kv head, KV split) over the query's chunk table (the selected groups'
page ranges, no assembled copy), with fp32 partials merged by K3m.

Torch is plumbing here (device memory, the current stream, cuBLAS GEMMs for
the dense projections); every attention / page / selection step is a kernel
of libdbsa_sm100a.so.  There is no CPU path: without CUDA this raises.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as nat
from . import ops
from .errors import ConfigError, ValidationError

PAGE = ops.PAGE
SEG_FULL, SEG_SELF = nat.SEG_FULL, nat.SEG_SELF


def m_tiles(rows_needed: int) -> int:
    """128-row M tiles per attention work: 2 (two ping-ponged M tiles, Q in
    smem) or 1 (one M tile, Q in TMEM, double-buffered S).  DBSA_ATTN_TILES
    forces one kind; the default takes two tiles whenever a slab has more than
    128 rows."""
    import os

    forced = os.environ.get("DBSA_ATTN_TILES")
    if forced in ("1", "2"):
        return int(forced)
    return 2 if rows_needed > 128 else 1


def _torch():
    import torch

    return torch


def default_device(device=None):
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2503_08640_b200 needs a CUDA (sm_100a) device; there is no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise RuntimeError(f"device {dev} is not a CUDA device; there is no CPU fallback")
    return dev if dev.index is not None else torch.device("cuda", torch.cuda.current_device())


# ============================================================== weights
class DeviceModel:
    """Weights resident in HBM, laid out for the fused projections:
    wqkv = [wq | wk | wv] (d, (H + 2 Hkv) hd) and wgu = [w_gate | w_up]
    (d, 2 ffn) as bf16 GEMM operands; lm_head K-major as lm_head_t
    (vocab, d), the B operand of K5 (the fused label scoring); embedding,
    norms and the residual stream stay fp32 (the reference's f32 storage,
    kernels.py:1-7)."""

    def __init__(self, config, device, embed, layers, out_norm, lm_head=None, lm_head_t=None):
        self.config = config
        self.device = device
        self.embed = embed
        self.layers = layers
        self.out_norm = out_norm
        self.lm_head_t = lm_head_t if lm_head_t is not None else lm_head.t().contiguous()
        self.rope = ops.rope_table(config.max_seq_len, config.head_dim, config.rope_theta, device)
        self.config_hash = config.hash_bytes()

    @classmethod
    def from_weights(cls, weights, device):
        torch = _torch()
        t = weights.tensors

        def f32(name):
            return torch.from_numpy(np.ascontiguousarray(t[name])).to(device)

        def bf(*names):
            arr = np.concatenate([t[n] for n in names], axis=1) if len(names) > 1 else t[names[0]]
            return torch.from_numpy(np.ascontiguousarray(arr)).to(device).to(torch.bfloat16)

        layers = []
        for i in range(weights.config.n_layers):
            p = f"layers.{i}."
            layers.append(dict(attn_norm=f32(p + "attn_norm"), wqkv=bf(p + "wq", p + "wk", p + "wv"),
                               wo=bf(p + "wo"), ffn_norm=f32(p + "ffn_norm"), wgu=bf(p + "w_gate", p + "w_up"),
                               wdown=bf(p + "w_down")))
        lm_t = torch.from_numpy(np.ascontiguousarray(t["lm_head"].T)).to(device).to(torch.bfloat16)
        return cls(weights.config, device, f32("tok_embed"), layers, f32("out_norm"), lm_head_t=lm_t)

    @classmethod
    def random(cls, config, seed: int = 0, device=None):
        """Device-side random init with the reference's scaled-uniform scheme
        (model.py:159-171): norms 1, embedding U(+-0.1), projections
        U(+-1/sqrt(fan_in)).  Used for the Llama-scale configurations whose
        float32 host copy would not be practical; not bit-identical to
        init_random's Philox stream."""
        torch = _torch()
        dev = default_device(device)
        g = torch.Generator(device=dev)
        g.manual_seed(int(seed))
        c = config
        qw, kw = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim

        def u(shape, fan_in, dtype=torch.bfloat16):
            b = 1.0 / math.sqrt(fan_in)
            return torch.empty(shape, dtype=dtype, device=dev).uniform_(-b, b, generator=g)

        ones = lambda n: torch.ones(n, dtype=torch.float32, device=dev)  # noqa: E731
        layers = [dict(attn_norm=ones(c.d_model), wqkv=u((c.d_model, qw + 2 * kw), c.d_model),
                       wo=u((qw, c.d_model), qw), ffn_norm=ones(c.d_model),
                       wgu=u((c.d_model, 2 * c.ffn_dim), c.d_model), wdown=u((c.ffn_dim, c.d_model), c.ffn_dim))
                  for _ in range(c.n_layers)]
        embed = torch.empty((c.vocab_size, c.d_model), dtype=torch.float32, device=dev).uniform_(-0.1, 0.1, generator=g)
        return cls(c, dev, embed, layers, ones(c.d_model), lm_head_t=u((c.vocab_size, c.d_model), c.d_model))

    @property
    def lm_head(self):
        """The reference's (d, vocab) lm_head, as a transposed view."""
        return self.lm_head_t.t()

    def rope_for(self, rows: int):
        """Rope table covering positions [0, rows) (stage 2 reads rows
        position - delta, which may exceed max_seq_len); grown on demand."""
        if rows > self.rope.shape[0]:
            self.rope = ops.rope_table(max(rows, 2 * self.rope.shape[0]), self.config.head_dim,
                                       self.config.rope_theta, self.device)
        return self.rope

    def nbytes(self) -> int:
        n = self.embed.numel() * 4 + self.lm_head_t.numel() * 2
        for lw in self.layers:
            n += sum(v.numel() * v.element_size() for v in lw.values())
        return n


# ============================================================== page store (K2)
class PageStore:
    """The cache's HBM page pool.  K [L][Hkv][rows][HDP], V^T [L][Hkv][HDP][rows]
    (bf16); rows are handed out in whole 64-token pages per group."""

    def __init__(self, config, device, capacity_tokens: int = 0):
        self.config = config
        self.device = device
        self.hdp = ops.hd_pad(config.head_dim)
        self.used_rows = 0
        self.rows = 0
        self.k = self.v = None
        self._rope = None
        if capacity_tokens:
            self._grow(_round_page(capacity_tokens) + PAGE)

    @property
    def rope(self):
        if self._rope is None:
            self._rope = ops.rope_table(self.config.max_seq_len, self.config.head_dim, self.config.rope_theta,
                                        self.device)
        return self._rope

    def _grow(self, rows: int) -> None:
        torch = _torch()
        c = self.config
        rows = _round_page(rows)
        k = torch.zeros((c.n_layers, c.n_kv_heads, rows, self.hdp), dtype=torch.bfloat16, device=self.device)
        v = torch.zeros((c.n_layers, c.n_kv_heads, self.hdp, rows), dtype=torch.bfloat16, device=self.device)
        if self.k is not None and self.used_rows:
            k[:, :, : self.used_rows].copy_(self.k[:, :, : self.used_rows])
            v[..., : self.used_rows].copy_(self.v[..., : self.used_rows])
        self.k, self.v, self.rows = k, v, rows

    def reserve(self, counts) -> list[int]:
        need = sum(_round_page(n) for n in counts)
        if self.used_rows + need > self.rows:
            self._grow(max(self.used_rows + need, self.rows + self.rows // 2))
        out = []
        for n in counts:
            out.append(self.used_rows)
            self.used_rows += _round_page(n)
        return out

    def nbytes(self) -> int:
        return 0 if self.k is None else 2 * self.k.numel() * 2

    def planes(self):
        return (self.k, self.v, self.rows, self.config.n_layers)

    def write_host_group(self, entry, pre_kv) -> None:
        """Upload one group's host pre-rotation K/V and write its pages (K2w)."""
        torch = _torch()
        c = self.config
        n = entry.token_count
        pos = torch.arange(entry.pos_start, entry.pos_end, dtype=torch.int32, device=self.device)
        pages = _pages_for([(0, n, entry.row0)])
        pdev = ops.to_device(pages, self.device)
        for layer, (k, v) in enumerate(pre_kv):
            ks = torch.from_numpy(np.ascontiguousarray(k, np.float32)).to(self.device).to(torch.bfloat16)
            vs = torch.from_numpy(np.ascontiguousarray(v, np.float32)).to(self.device).to(torch.bfloat16)
            ops.kv_write(ks.reshape(n, -1), vs.reshape(n, -1), c.n_kv_heads * c.head_dim, pos, self.rope, pdev,
                         len(pages), self.k, self.v, self.rows, c.n_layers, layer, c.n_kv_heads, c.head_dim)
        torch.cuda.current_stream(self.device).synchronize()

    def read_rows(self, layer: int, row0: int, n: int):
        """(K rotated, V) float32 (n, Hkv, hd) of a row range (host copy)."""
        hd = self.config.head_dim
        k = self.k[layer, :, row0:row0 + n, :hd].float().permute(1, 0, 2).cpu().numpy()
        v = self.v[layer, :, :hd, row0:row0 + n].float().permute(2, 0, 1).cpu().numpy()
        return np.ascontiguousarray(k), np.ascontiguousarray(v)


def _round_page(n: int) -> int:
    return -(-int(n) // PAGE) * PAGE


def _pages_for(spans) -> np.ndarray:
    """spans: (first token in the source buffer, n_tok, first destination row)."""
    out = []
    for tok0, n, row0 in spans:
        for i in range(0, n, PAGE):
            out.append((tok0 + i, min(PAGE, n - i), row0 + i, 0))
    return np.array(out, dtype=np.int32).reshape(-1, 4).view(ops.PAGE_DTYPE).reshape(-1)


def _seg_array(segs) -> np.ndarray:
    a = np.zeros(len(segs), dtype=ops.SEG_DTYPE)
    if segs:
        s = np.asarray(segs, dtype=np.int32).reshape(len(segs), -1)
        for i, name in enumerate(("src", "layer", "row0", "n_tok", "kind", "shift")):
            a[name] = s[:, i]
    return a


def _per_layer_segs(seg_arr: np.ndarray, n_layers: int) -> np.ndarray:
    """[L, n_segs]: pool segments (src 0) address layer l, aux (src 1) layer 0."""
    out = np.repeat(seg_arr[None, :], n_layers, axis=0)
    pool = out["src"] == 0
    out["layer"] = np.where(pool, np.arange(n_layers, dtype=np.int32)[:, None], 0)
    return out


def _work_array(works) -> np.ndarray:
    a = np.zeros(len(works), dtype=ops.WORK_DTYPE)
    if works:
        w = np.asarray(works, dtype=np.int64).reshape(len(works), -1)
        for i, name in enumerate(ops.WORK_DTYPE.names):
            a[name] = w[:, i]
    return a


# ============================================================== dense block
def mm_f32(a, b, out):
    """out (fp32) = a @ b for bf16 operands, fp32 accumulate and output (cuBLAS)."""
    torch = _torch()
    try:
        return torch.mm(a, b, out_dtype=torch.float32, out=out)
    except (TypeError, RuntimeError):
        out.copy_(torch.mm(a, b, out_dtype=torch.float32))
        return out


class _Scratch:
    """Per-forward activation buffers, reused across layers."""

    def __init__(self, dm, n_tok):
        torch = _torch()
        c, dev = dm.config, dm.device
        qw, kw = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
        self.x = torch.empty((n_tok, c.d_model), dtype=torch.bfloat16, device=dev)
        self.qkv = torch.empty((n_tok, qw + 2 * kw), dtype=torch.bfloat16, device=dev)
        self.att = torch.empty((n_tok, qw), dtype=torch.bfloat16, device=dev)
        self.proj = torch.empty((n_tok, c.d_model), dtype=torch.float32, device=dev)
        self.ffn_chunk = max(1, min(n_tok, (1 << 31) // (2 * c.ffn_dim * 2)))
        self.gu = torch.empty((min(n_tok, self.ffn_chunk), 2 * c.ffn_dim), dtype=torch.bfloat16, device=dev)
        self.act = torch.empty((min(n_tok, self.ffn_chunk), c.ffn_dim), dtype=torch.bfloat16, device=dev)


def _decoder_gen(dm, ids_dev, attend, write_kv, n_layers=None, kv_only_last=False, keep_last=None,
                 attend_early=None):
    """Pre-norm decoder body (model.py:319-359) over n new tokens, as a
    generator: it yields after each layer's `write_kv(l, qkv)` (the point where
    a multi-shard caller exchanges pages) and returns the fp32 final hidden
    states.  `attend(l, qkv, out)` fills the attention output.  kv_only_last:
    the caller only keeps K/V (a pool encode): the last layer stops after its
    page write -- its attention, O projection and FFN feed nothing -- and the
    return value is None.  keep_last (device int64 row indices): only those rows'
    outputs are used (the scored rows of a label batch), so the last layer's O
    projection and FFN run on them alone and the returned hidden states are
    those rows, in keep_last order.  attend_early(l, qkv, out), when given,
    runs right after the page write, before the yield (the part of the
    attention that does not wait for the caller's page exchange)."""
    torch = _torch()
    c = dm.config
    n = ids_dev.shape[0]
    s = _Scratch(dm, n)
    h = dm.embed.index_select(0, ids_dev)
    L = c.n_layers if n_layers is None else n_layers
    for layer in range(L):
        lw = dm.layers[layer]
        if layer == 0:
            ops.rmsnorm(h, lw["attn_norm"], c.norm_eps, out=s.x)
        else:  # the previous layer's FFN residual add, fused with this norm
            ops.add_rmsnorm(h, s.proj, lw["attn_norm"], c.norm_eps, s.x)
        torch.mm(s.x, lw["wqkv"], out=s.qkv)
        write_kv(layer, s.qkv)
        last_kv_only = kv_only_last and layer == L - 1
        if attend_early is not None and not last_kv_only:
            attend_early(layer, s.qkv, s.att)
        yield layer
        if last_kv_only:
            return None
        compact = attend(layer, s.qkv, s.att)
        if keep_last is not None and layer == L - 1:
            k = keep_last.numel()
            # attend() may have produced the kept rows alone, back to back (Stage2Plan.last)
            att = s.att[:k] if compact else s.att.index_select(0, keep_last)
            h = h.index_select(0, keep_last)
            proj, xk = s.proj[:k], s.x[:k]
            mm_f32(att, lw["wo"], proj)
            ops.add_rmsnorm(h, proj, lw["ffn_norm"], c.norm_eps, xk)
            for a in range(0, k, s.ffn_chunk):
                b = min(k, a + s.ffn_chunk)
                gu, act = s.gu[: b - a], s.act[: b - a]
                torch.mm(xk[a:b], lw["wgu"], out=gu)
                ops.silu_mul(gu, c.ffn_dim, out=act)
                mm_f32(act, lw["wdown"], proj[a:b])
            h.add_(proj)
            return h
        mm_f32(s.att, lw["wo"], s.proj)
        ops.add_rmsnorm(h, s.proj, lw["ffn_norm"], c.norm_eps, s.x)
        for a in range(0, n, s.ffn_chunk):
            b = min(n, a + s.ffn_chunk)
            gu, act = s.gu[: b - a], s.act[: b - a]
            torch.mm(s.x[a:b], lw["wgu"], out=gu)
            ops.silu_mul(gu, c.ffn_dim, out=act)
            mm_f32(act, lw["wdown"], s.proj[a:b])
    if L:
        h.add_(s.proj)
    return h


def _drain(gen):
    try:
        while True:
            next(gen)
    except StopIteration as e:
        return e.value


def _decoder(dm, ids_dev, attend, write_kv, n_layers=None, keep_last=None):
    return _drain(_decoder_gen(dm, ids_dev, attend, write_kv, n_layers, keep_last=keep_last))


# ============================================================== stage 1 (K1 + K2w)
class Stage1Plan:
    """Device tables of one layer-synchronous stage-1 encode of groups
    `new` (BlockEntry list; their tokens are contiguous, first at tok_base)."""

    def __init__(self, dm, cache, new, pattern, late_blocks=None):
        """late_blocks: groups whose pages of each layer arrive by the halo
        exchange (encode_pool_sharded).  The works that read one of them go
        last (`n_early` works before them), so the rest can run while the
        exchange is in flight."""
        c = dm.config
        gs, hkv = c.group_size, c.n_kv_heads
        late_blocks = set(late_blocks or ())
        # token buffer = the listed groups' tokens back to back (groups need not be contiguous)
        local_of = {}
        acc = 0
        for e in new:
            local_of[e.block_id] = acc
            acc += e.token_count
        self.n_tok = acc
        longest = max(e.token_count for e in new)
        self.num_m = m_tiles(longest * gs)
        slab = (128 * self.num_m) // gs
        if slab < 1:
            raise ConfigError(f"group size {gs} exceeds the 256 rows of one K1 work")
        segs, works = [], []
        pairs = 0
        for e in new:
            ctx = [cache.blocks[j] for j in pattern.context_of(e.block_id)]
            n_ctx = sum(x.token_count for x in ctx)
            local0 = local_of[e.block_id]
            t = e.token_count
            pairs += n_ctx * t + t * (t + 1) // 2
            for t0 in range(0, t, slab):
                nt = min(slab, t - t0)
                sb = len(segs)
                segs += [(0, 0, x.row0, x.token_count, SEG_FULL, 0) for x in ctx]
                segs.append((0, 0, e.row0, t0 + nt, SEG_SELF, 0))
                keys = n_ctx + t0 + nt
                for kv in range(hkv):
                    works.append((keys, local0 + t0, nt, local0, kv, sb, len(segs), 0, 0, 0))
        # Group-major order: the slabs x kv heads of one group run together, so its
        # context groups are read from HBM once and re-read from L2; among groups,
        # the longest key streams go first (shorter tail wave).
        longest = {}
        for wk in works:
            longest[wk[3]] = max(longest.get(wk[3], 0), wk[0])
        late_groups = {local_of[e.block_id] for e in new
                       if late_blocks & set(pattern.context_of(e.block_id))}
        works.sort(key=lambda wk: (wk[3] in late_groups, -longest[wk[3]], wk[3], -wk[0]))
        self.n_early = sum(1 for wk in works if wk[3] not in late_groups)
        self.pairs = pairs
        self.n_works = len(works)
        self.n_segs = len(segs)
        self.keys_visited = sum(w[0] * w[2] * gs for w in works)
        dev = dm.device
        self.works = ops.to_device(_work_array([w[1:] for w in works]), dev)
        self.segs = ops.to_device(_per_layer_segs(_seg_array(segs), c.n_layers), dev)
        pages = _pages_for([(local_of[e.block_id], e.token_count, e.row0) for e in new])
        self.n_pages = len(pages)
        self.pages = ops.to_device(pages, dev)
        torch = _torch()
        pos = np.concatenate([np.arange(e.pos_start, e.pos_end, dtype=np.int32) for e in new])
        self.pos = torch.from_numpy(pos).to(dev, non_blocking=True)

    def segs_ptr(self, layer: int) -> int:
        return self.segs.data_ptr() + layer * self.n_segs * ops.SEG_DTYPE.itemsize


def encode_groups_gen(dm, cache, new, ids, pattern, layers=None, late_blocks=None, kv_written=None):
    """Stage 1 for groups `new` (BlockEntry list) whose concatenated token ids
    are `ids`, as a generator pausing after each layer's page write (see
    _decoder_gen).  Returns the attended pair count of these groups
    (pipeline.py:231-232) as COUNTED BY K1: layer 0's launch adds every
    (row, key) pair that entered its softmax (DbsaAttnArgs.pair_count), all
    heads; that total must equal n_heads x the plan's pair count
    (masks.count_allowed_token_pairs, masks.py:111-123), else the kernel
    visited a wrong tile set and this raises."""
    torch = _torch()
    c = dm.config
    plan = Stage1Plan(dm, cache, new, pattern, late_blocks)
    n_layers = c.n_layers if layers is None else layers
    counter = torch.zeros(1, dtype=torch.int64, device=dm.device) if n_layers > 1 else None
    store = cache.store
    qw, kw = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
    stride = qw + 2 * kw
    ids_dev = torch.as_tensor(np.asarray(ids, dtype=np.int64)).to(dm.device, non_blocking=True)

    def write_kv(layer, qkv):
        ops.kv_write(qkv[:, qw:], qkv[:, qw + kw:], stride, plan.pos, dm.rope, plan.pages, plan.n_pages, store.k,
                     store.v, store.rows, c.n_layers, layer, c.n_kv_heads, c.head_dim)
        if kv_written is not None:  # the halo exchange of this layer may start here
            kv_written(layer)

    def launch(layer, qkv, out, w0, w1, after_kv_write):
        if w1 > w0:
            ops.attention(q=qkv, q_tok_stride=stride, tok_pos=plan.pos, tok_lo=None, rope=dm.rope,
                          pool=store.planes(), aux=None, n_heads=c.n_heads, n_kv_heads=c.n_kv_heads,
                          head_dim=c.head_dim, works_dev=plan.works.data_ptr() + w0 * ops.WORK_DTYPE.itemsize,
                          n_works=w1 - w0, segs_dev=plan.segs_ptr(layer), num_m=plan.num_m, out=out,
                          out_tok_stride=qw, pair_count=counter if layer == 0 else None,
                          after_kv_write=after_kv_write)

    n_early = plan.n_early if late_blocks else 0  # without a halo every work runs in attend()

    def attend_early(layer, qkv, out):  # works that read no halo group: before the exchange
        launch(layer, qkv, out, 0, n_early, True)

    def attend(layer, qkv, out):  # the rest, once the layer's halo pages are in
        launch(layer, qkv, out, n_early, plan.n_works, n_early == 0)

    # only the pages are kept: the last layer's attention / O / FFN are skipped
    yield from _decoder_gen(dm, ids_dev, attend, write_kv, n_layers=layers, kv_only_last=True,
                            attend_early=attend_early if late_blocks else None)
    if counter is None:  # a one-layer model runs no attention in stage 1 (its output feeds nothing)
        return plan.pairs
    visited = int(counter.item())
    if visited != plan.pairs * c.n_heads:
        raise RuntimeError(f"K1 visited {visited} (row, key) pairs, expected n_heads x {plan.pairs}")
    return visited // c.n_heads


def encode_groups(dm, cache, new, ids, pattern, layers=None) -> int:
    """Stage 1 for groups `new` on one device; returns attended pairs."""
    return _drain(encode_groups_gen(dm, cache, new, ids, pattern, layers))


def encode_pool_sharded(dm, blocks, pattern, comm, device=None):
    """Group-sharded stage 1: the groups are split into
    contiguous ranges, every rank re-encodes the sink, and per layer the K/V
    pages its successors need travel as a halo (parallel.exchange_pages).

    blocks: [(token ids, sha256 digest, demo spans)] of the whole pool.
    Returns ({local rank: SegmentedKVCache holding that rank's groups, the sink
    and its halo}, attended pairs of the local ranks' own groups, ranges).
    """
    from . import parallel
    from .kvstore import SegmentedKVCache

    c = dm.config
    counts = [len(ids) for ids, _, _ in blocks]
    n_blocks = len(blocks)
    ranges = parallel.plan_group_shards(counts, comm.world)
    halo = parallel.halo_plan(pattern, ranges, n_blocks)
    caches, gens = {}, {}
    torch = _torch()
    dev = torch.device(device) if device is not None else dm.device
    # the halo exchange runs on a side stream that waits only for the layer's
    # page writes; the K1 works that read no halo group run meanwhile
    side = torch.cuda.Stream(dev) if dev.type == "cuda" else None
    kv_events = {}

    def on_kv_written(r):
        def record(layer):
            if side is not None:
                ev = torch.cuda.Event()
                ev.record()
                kv_events[r] = ev
        return record

    for r in comm.local_ranks:
        present = parallel.local_groups(pattern, ranges, r, n_blocks)
        # page-rounded capacity: reserve() must not grow (a second buffer while the first lives)
        cache = SegmentedKVCache(c, device or dm.device, capacity_tokens=sum(_round_page(counts[g]) for g in present))
        cache._reserve_subset(counts, [d for _, d, _ in blocks], [sp for _, _, sp in blocks], present)
        compute = sorted({0} | set(range(*ranges[r])))
        new = [cache.blocks[g] for g in compute]
        ids = np.concatenate([np.asarray(blocks[g][0], np.int64) for g in compute])
        caches[r] = cache
        gens[r] = encode_groups_gen(dm, cache, new, ids, pattern,
                                    late_blocks={g for g, _, dst in halo if dst == r},
                                    kv_written=on_kv_written(r))
    pairs = {}
    stores = {r: caches[r].store for r in caches}
    entries = {r: {e.block_id: e for e in caches[r].blocks if e.row0 >= 0} for r in caches}
    for layer in range(c.n_layers):
        for r in caches:
            next(gens[r])
        if side is None:
            parallel.exchange_pages(comm, layer, halo, stores, entries)
            continue
        for ev in kv_events.values():
            side.wait_event(ev)
        with torch.cuda.stream(side):
            parallel.exchange_pages(comm, layer, halo, stores, entries)
        torch.cuda.current_stream(dev).wait_stream(side)
    for r in caches:
        pairs[r] = _drain(gens[r])
        if r != 0:  # the sink's own pairs are counted once, on rank 0
            t0 = counts[0]
            pairs[r] -= t0 * (t0 + 1) // 2
    for cache in caches.values():
        cache.seal()
    return caches, pairs, ranges


# ============================================================== stage 2 (K3 + K3m)
class QueryJob:
    """One stage-2 forward: new tokens (query, then label branches) against a
    chunk table.  pos/lo are LOCAL (position = n_ctx + pos; lo = lowest
    non-prefix self key visible, tree mask).  `labels` (label token lists)
    is set for label-scoring jobs."""

    __slots__ = ("chunks", "n_ctx", "ids", "pos", "lo", "prefix", "labels")

    def __init__(self, chunks, n_ctx, ids, pos, lo, prefix, labels=None):
        self.chunks, self.n_ctx, self.ids, self.pos, self.lo, self.prefix = chunks, n_ctx, ids, pos, lo, prefix
        self.labels = labels


def label_job(chunks, n_ctx, query_ids, labels) -> QueryJob:
    """Query followed by every label as a branch of a token tree.

    The LAST token of each label is not fed: its logits are never scored
    (score_label reads rows len(q)-1 .. len(q)+len(label)-2, model.py:441-443)
    and no other token attends to it (it ends its branch), so dropping it
    leaves every label score unchanged."""
    nq = len(query_ids)
    ids, pos, lo = list(query_ids), list(range(nq)), [0] * nq
    for lab in labels:
        start = len(ids)
        fed = list(lab)[:-1]
        ids += fed
        pos += list(range(nq, nq + len(fed)))
        lo += [start] * len(fed)
    return QueryJob(chunks, n_ctx, ids, pos, lo, nq, [list(x) for x in labels])


def pad_job(job: QueryJob, n_tok: int, max_seq_len: int) -> QueryJob:
    """`job` with dummy tokens appended up to n_tok new tokens: one more tree
    branch after the labels (positions after the job's last, visible to
    nothing but itself), so every real token's keys, outputs and label scores
    are unchanged; only the launch shape is.  Returned as is when already
    long enough or when the padding would pass max_seq_len."""
    d = n_tok - len(job.ids)
    if d <= 0:
        return job
    p0 = max(job.pos) + 1
    if job.n_ctx + p0 + d > max_seq_len:
        return job
    start = len(job.ids)
    return QueryJob(job.chunks, job.n_ctx, list(job.ids) + [0] * d, list(job.pos) + list(range(p0, p0 + d)),
                    list(job.lo) + [start] * d, job.prefix, job.labels)


class NewTokens:
    """The new (query / label) tokens of a stage-2 batch: ids, rotary positions,
    tree bounds and their K/V pages (one aux page set, page-aligned per job)."""

    def __init__(self, dm, jobs):
        torch = _torch()
        c = dm.config
        gs = c.group_size
        self.n_jobs = len(jobs)
        self.n_new = [len(j.ids) for j in jobs]
        self.tok0 = np.concatenate([[0], np.cumsum(self.n_new)]).astype(np.int64)
        self.n_tok = int(self.tok0[-1])
        self.num_m = m_tiles(max(self.n_new) * gs)
        self.slab = (128 * self.num_m) // gs
        if self.slab < 1:
            raise ConfigError(f"group size {gs} exceeds the 256 rows of one K3 work")
        # balanced slabs: ceil(n / slab) pieces of equal size (e.g. 44 tokens -> 22 + 22
        # rather than 32 + 12 at one M tile, so no work is mostly padding)
        self.slabs = []
        for n in self.n_new:
            k = -(-n // self.slab)
            size = -(-n // k)
            self.slabs.append([(t0, min(size, n - t0)) for t0 in range(0, n, size)])
        self.aux_row0 = np.concatenate([[0], np.cumsum([_round_page(n) for n in self.n_new])]).astype(np.int64)
        self.aux_rows = int(self.aux_row0[-1])
        dev = dm.device
        pos = np.concatenate([np.asarray(j.pos, np.int64) + j.n_ctx for j in jobs]).astype(np.int32)
        lo = np.concatenate([np.asarray(j.lo, np.int64) for j in jobs]).astype(np.int32)
        ids = np.concatenate([np.asarray(j.ids, np.int64) for j in jobs])
        if int(pos.max()) >= c.max_seq_len:
            raise ValidationError(f"position {int(pos.max())} exceeds max_seq_len {c.max_seq_len}")
        self.max_pos = int(pos.max())
        self.pos_host = pos
        self.pos = ops.h2d(pos, dev)
        self.lo = ops.h2d(lo, dev)
        self.ids = ops.h2d(ids, dev)
        self.pages = ops.to_device(_pages_for([(int(self.tok0[i]), self.n_new[i], int(self.aux_row0[i]))
                                               for i in range(len(jobs))]), dev)
        self.n_pages = int(sum(-(-n // PAGE) for n in self.n_new))
        self._aux_shape = (c.n_kv_heads, ops.hd_pad(c.head_dim), dev)
        self._aux = None
        # canonical partial layout (sharded mode): one row block per (job, slab, kv head)
        self.part_base = []
        base = 0
        for qi in range(len(jobs)):
            per = []
            for t0, nt in self.slabs[qi]:
                per.append(base)
                base += nt * gs * c.n_kv_heads
            self.part_base.append(per)
        self.canon_rows = base

    def _aux_planes(self):
        # allocated on first use: a batch that replays a captured graph writes the
        # graph's own aux pages, never these
        if self._aux is None:
            torch = _torch()
            hkv, hdp, dev = self._aux_shape
            self._aux = (torch.zeros((1, hkv, self.aux_rows, hdp), dtype=torch.bfloat16, device=dev),
                         torch.zeros((1, hkv, hdp, self.aux_rows), dtype=torch.bfloat16, device=dev))
        return self._aux

    @property
    def k_aux(self):
        return self._aux_planes()[0]

    @property
    def v_aux(self):
        return self._aux_planes()[1]

    def aux(self):
        return (self.k_aux, self.v_aux, self.aux_rows, 1)


# Split-KV table templates (AttnSchedule), LRU, per thread: a template's device
# tables are then only ever used on that thread's stream (Runner.infer gives
# each thread its own), so eviction cannot free a block another stream reads.
_SPLIT_TLS = __import__("threading").local()
_SPLIT_TEMPLATES_MAX = 64


def _split_templates():
    d = getattr(_SPLIT_TLS, "cache", None)
    if d is None:
        d = _SPLIT_TLS.cache = __import__("collections").OrderedDict()
    return d


def _split_bf16() -> bool:
    """Split-KV partials in bf16 (as the chunk-major ones): half the epilogue
    and K3m bytes of a latency launch; DBSA_SPLIT_BF16=0 keeps fp32."""
    import os

    return os.environ.get("DBSA_SPLIT_BF16", "1") == "1"


def _split_cm() -> bool:
    # DBSA_SPLIT_CM=0: split-KV launches keep the generic kernel instance
    import os

    return os.environ.get("DBSA_SPLIT_CM", "1") != "0"


class AttnSchedule:
    """K3 works + segments (+ K3m merge groups) of a batch against chunk tables.

    mode "split": each (job, kv head, slab) is cut into splits over its chunks
    (split-KV for parallelism); partials of multi-split works merge in place.
    mode "canonical": exactly one work per (job, kv head, slab) that has any
    key on this shard, always writing an fp32 partial + LSE at the canonical
    row block (NewTokens.part_base) -- the per-rank half of the C5 merge.
    include_self: whether this schedule covers the jobs' own tokens (SELF).
    """

    def __init__(self, dm, jobs, nt: NewTokens, chunk_tables=None, target_ctas=None, order="query",
                 mode="split", include_self=True, pack=None):
        torch = _torch()
        c = dm.config
        gs, hkv, hd = c.group_size, c.n_kv_heads, c.head_dim
        tables = chunk_tables if chunk_tables is not None else [j.chunks for j in jobs]
        target = target_ctas or 4 * 148
        # pack: SELF becomes a split of its own and the works are packed onto the
        # CTAs by cost (pack_works), instead of SELF riding on the last chunk
        # split and round-robin placement (the one-wave tail of a latency launch)
        if pack is None:
            import os

            pack = mode == "split" and nt.num_m == 2 and os.environ.get("DBSA_PACK", "1") != "0"
        self.pack = pack
        dev = dm.device
        # split-KV tables depend on the chunk LENGTHS (and page offsets), not on
        # which groups were picked: a cached template is refilled with this
        # batch's chunk rows and shifts (the batch-1 planning cost of Runner.infer)
        key = None
        if mode == "split" and order == "query":
            key = (tuple(tuple((int(r[1]), int(r[0]) % PAGE) for r in np.asarray(t, np.int64).reshape(-1, 3))
                         for t in tables),
                   tuple(int(x) for x in nt.n_new), tuple(int(j.prefix) for j in jobs), nt.num_m, include_self,
                   pack, target, gs, hkv, hd, c.n_layers, str(dev), _split_bf16())
            templates = _split_templates()
            tpl = templates.get(key)
            if tpl is not None:
                templates.move_to_end(key)
                self._from_template(dm, nt, tables, tpl)
                return
        segs, works, merges = [], [], []
        seg_src = []  # per segment: (job, chunk index) or (job, -1) for SELF
        min_shift = 0
        part_rows = 0 if mode == "split" else nt.canon_rows
        kv_tok = 0
        for qi, j in enumerate(jobs):
            n = nt.n_new[qi]
            slabs = nt.slabs[qi]
            ch = np.asarray(tables[qi], dtype=np.int64).reshape(-1, 3)
            kv_tok += int(ch[:, 1].sum()) if len(ch) else 0
            chunk_segs = []
            for row, cnt, delta in ch:
                # queries of this chunk use rope row (position - delta)
                chunk_segs.append((0, 0, int(row), int(cnt), SEG_FULL, int(delta)))
                min_shift = min(min_shift, int(delta))
            q0 = int(nt.tok0[qi])
            if mode == "canonical":
                if not chunk_segs and not include_self:
                    continue
                for si, (t0, ntk) in enumerate(slabs):
                    rows = ntk * gs
                    sb = len(segs)
                    segs += chunk_segs
                    if include_self:
                        segs.append((1, 0, int(nt.aux_row0[qi]), t0 + ntk, SEG_SELF, 0))
                    for kv in range(hkv):
                        works.append((q0 + t0, ntk, q0, kv, sb, len(segs), j.prefix, 1,
                                      nt.part_base[qi][si] + kv * rows))
                continue
            n_split = max(1, min(len(ch), -(-target // max(1, len(jobs) * hkv * len(slabs)))))
            bounds = _split_bounds(ch[:, 1] if len(ch) else np.zeros(0, np.int64), n_split)
            split_ranges = []
            own_self = self.pack and include_self and len(ch) > 0
            for sp in range(n_split - 1 + own_self):
                sb = len(segs)
                segs += chunk_segs[bounds[sp]:bounds[sp + 1]]
                seg_src += [(qi, u) for u in range(bounds[sp], bounds[sp + 1])]
                split_ranges.append((sb, len(segs)))
            n_split += own_self
            for t0, ntk in slabs:
                rows = ntk * gs
                last_sb = len(segs)
                if not own_self:
                    segs += chunk_segs[bounds[n_split - 1]:bounds[n_split]]
                    seg_src += [(qi, u) for u in range(bounds[n_split - 1], bounds[n_split])]
                if include_self:
                    segs.append((1, 0, int(nt.aux_row0[qi]), t0 + ntk, SEG_SELF, 0))
                    seg_src.append((qi, -1))
                last = (last_sb, len(segs))
                for kv in range(hkv):
                    base = part_rows
                    mode_w = 1 if n_split > 1 else 0
                    for sp in range(n_split):
                        sb, se = last if sp == n_split - 1 else split_ranges[sp]
                        works.append((q0 + t0, ntk, q0, kv, sb, se, j.prefix, mode_w, base + sp * rows))
                    if n_split > 1:
                        merges.append((base, rows, n_split, q0 + t0, kv))
                        part_rows += n_split * rows
        if order == "chunk":
            first_row = [segs[wk[4]][2] if wk[5] > wk[4] and segs[wk[4]][0] == 0 else 1 << 30 for wk in works]
            idx = sorted(range(len(works)), key=lambda i: (first_row[i], works[i][3]))
            works = [works[i] for i in idx]
        self.cta_works, self.n_ctas = None, 0
        if self.pack and works:
            works, bounds_cta = pack_works(works, segs, _num_sms(dm.device))
            self.n_ctas = len(bounds_cta) - 1
            self.cta_works = ops.to_device(np.asarray(bounds_cta, dtype=np.int32), dm.device)
        self.kv_tokens = kv_tok
        self.n_works, self.n_segs, self.n_merge = len(works), len(segs), len(merges)
        # every work one segment, writing a partial (e.g. batch-1 packed splits):
        # the launch may use the specialised kernel instance (one_seg_partials)
        self.one_seg = _split_cm() and bool(works) and all(w[5] - w[4] == 1 and w[7] != 0 for w in works)
        self.works = ops.to_device(_work_array(works), dev)
        seg_arr = _seg_array(segs)
        self.segs = ops.to_device(_per_layer_segs(seg_arr, c.n_layers), dev)
        self.merges = ops.to_device(_merge_array(merges), dev) if merges else None
        self.max_rows = max((m[1] for m in merges), default=0)
        self.rope = dm.rope_for(nt.max_pos - min_shift + 1)
        self.part_rows = part_rows
        bf16 = mode == "split" and _split_bf16()
        self._part_spec = (max(part_rows, 1), hd, torch.bfloat16 if bf16 else torch.float32, dev)
        self._part = None
        if key is not None:
            src = np.asarray(seg_src, np.int64).reshape(-1, 2)
            templates = _split_templates()
            templates[key] = dict(
                works=self.works, merges=self.merges, cta_works=self.cta_works, n_ctas=self.n_ctas, segs=seg_arr,
                one_seg=self.one_seg,
                seg_job=src[:, 0], seg_chunk=src[:, 1], n_works=self.n_works, n_merge=self.n_merge,
                max_rows=self.max_rows, part_rows=part_rows, kv_tokens=kv_tok, part_dtype=self._part_spec[2])
            while len(templates) > _SPLIT_TEMPLATES_MAX:
                templates.popitem(last=False)

    def _from_template(self, dm, nt, tables, tpl):
        """This batch's split-KV tables from a cached template: the works, merge
        groups and CTA ranges as they are; the segments refilled with the
        batch's chunk rows and RoPE shifts and its own tokens' aux rows."""
        torch = _torch()
        c = dm.config
        segs = tpl["segs"].copy()
        job, chunk = tpl["seg_job"], tpl["seg_chunk"]
        tabs = [np.asarray(t, np.int64).reshape(-1, 3) for t in tables]
        allch = np.concatenate(tabs) if tabs else np.zeros((0, 3), np.int64)
        off = np.concatenate([[0], np.cumsum([len(t) for t in tabs])])
        full = chunk >= 0
        idx = off[job[full]] + chunk[full]
        segs["row0"][full] = allch[idx, 0]
        segs["shift"][full] = allch[idx, 2]
        segs["row0"][~full] = np.asarray(nt.aux_row0, np.int64)[job[~full]]
        min_shift = min(0, int(allch[:, 2].min())) if len(allch) else 0
        self.works, self.merges, self.cta_works, self.n_ctas = tpl["works"], tpl["merges"], tpl["cta_works"], tpl["n_ctas"]
        self.one_seg = tpl["one_seg"]
        self.n_works, self.n_segs, self.n_merge = tpl["n_works"], len(segs), tpl["n_merge"]
        self.segs = ops.to_device(_per_layer_segs(segs, c.n_layers), dm.device)
        self.max_rows, self.part_rows, self.kv_tokens = tpl["max_rows"], tpl["part_rows"], tpl["kv_tokens"]
        self.rope = dm.rope_for(nt.max_pos - min_shift + 1)
        self._part_spec = (max(self.part_rows, 1), c.head_dim, tpl["part_dtype"], dm.device)
        self._part = None

    def _partials(self):
        # allocated on first use: a batch that replays a captured graph uses the graph's
        if self._part is None:
            torch = _torch()
            n, hd, dt, dev = self._part_spec
            self._part = (torch.empty((n, hd), dtype=dt, device=dev), torch.empty((n,), dtype=torch.float32, device=dev))
        return self._part

    @property
    def part_o(self):
        return self._partials()[0]

    @part_o.setter
    def part_o(self, v):
        self._part = (v, self._partials()[1])

    @property
    def part_lse(self):
        return self._partials()[1]

    def segs_ptr(self, layer: int) -> int:
        return self.segs.data_ptr() + layer * self.n_segs * ops.SEG_DTYPE.itemsize

    def launch(self, dm, nt: NewTokens, layer, qkv, out, pool, part_o=None, part_lse=None):
        c = dm.config
        qw, kw = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
        if self.n_works == 0:
            return
        ops.attention(q=qkv, q_tok_stride=qw + 2 * kw, tok_pos=nt.pos, tok_lo=nt.lo, rope=self.rope,
                      pool=pool, aux=nt.aux(), n_heads=c.n_heads, n_kv_heads=c.n_kv_heads, head_dim=c.head_dim,
                      works_dev=self.works, n_works=self.n_works, segs_dev=self.segs_ptr(layer), num_m=nt.num_m,
                      out=out, out_tok_stride=qw, part_o=self.part_o if part_o is None else part_o,
                      part_lse=self.part_lse if part_lse is None else part_lse, cta_works=self.cta_works,
                      n_ctas=self.n_ctas, after_kv_write=True, one_seg_partials=self.one_seg)


# Cost model of pack_works, in key tiles: a CTA's first work pays the cold
# start (first Q staging, first-tile and epilogue code fetch: ~15 tiles of
# batch-1 K3 time, profiles/r02f_b1_tiles.txt), later works the warm work
# boundary (Q staging, drain, epilogue: ~5 tiles).
PACK_FIRST, PACK_NEXT = 15, 5


def pack_works(works, segs, n_sms: int):
    """Longest-processing-time packing of K3 works onto at most n_sms CTAs
    under the PACK_FIRST / PACK_NEXT cost model.  Returns the works reordered
    so each CTA's are contiguous (longest first) and the [n_ctas + 1] prefix
    offsets (DbsaAttnArgs.cta_works)."""
    import heapq

    sg = np.asarray(segs, dtype=np.int64).reshape(len(segs), -1)
    seg_tiles = (sg[:, 2] % PAGE + sg[:, 3] + 127) // 128 if len(sg) else np.zeros(0, np.int64)
    cum = np.concatenate([[0], np.cumsum(seg_tiles)])
    w = np.asarray(works, dtype=np.int64).reshape(len(works), -1)
    tiles = cum[w[:, 5]] - cum[w[:, 4]]
    order = np.argsort(-tiles, kind="stable")
    n_ctas = min(n_sms, len(works))
    # the n_ctas longest works open one CTA each; the rest go to the least loaded
    per_cta = [[int(i)] for i in order[:n_ctas]]
    heap = [(PACK_FIRST + int(tiles[i]), b) for b, i in enumerate(order[:n_ctas])]
    heapq.heapify(heap)
    for i in order[n_ctas:]:
        load, b = heap[0]
        heapq.heapreplace(heap, (load + PACK_NEXT + int(tiles[i]), b))
        per_cta[b].append(int(i))
    out, bounds = [], [0]
    for lst in per_cta:
        out += [works[i] for i in lst]
        bounds.append(len(out))
    return out, bounds


def _num_sms(device) -> int:
    torch = _torch()
    return torch.cuda.get_device_properties(device).multi_processor_count if device.type == "cuda" else 148


class ChunkMajorSchedule:
    """Chunk-major K3 for a BATCH of queries: one work stacks the rows of many
    queries against ONE selected chunk (DBSA_OUT_MAPPED works through a row
    map), so a chunk's K/V tiles are streamed once per 128*num_m rows instead
    of once per query, and the MMA M tiles are full instead of holding one
    query's gs * n_new rows (176 of 256 at C3).  Every (query, chunk) pair and
    every query's own tokens (SELF, per-query works) produce an fp32 partial +
    LSE; K3m merges the S_q = n_chunks + 1 partials of each query row -- the
    single softmax over the concatenated key set of kernels.py:52-56.

    Partial layout, per kv head: [query][split s][token][gs] rows (split s of
    query q = its s-th chunk, the last split = SELF), so a query's merge group
    is (base, rows = n * gs, n_splits = S_q) with the default split stride.
    The RoPE re-positioning delta of (query, chunk) is folded into each map
    entry's rope row (tok_pos - delta)."""

    def __init__(self, dm, jobs, nt: NewTokens, chunk_tables=None, num_m: int = 2, include_self: bool = True,
                 subsets=None):
        torch = _torch()
        c = dm.config
        hd = c.head_dim
        tables = chunk_tables if chunk_tables is not None else [j.chunks for j in jobs]
        self.num_m = num_m
        t = chunk_major_tables(tables, nt.n_new, nt.pos_host, nt.aux_row0, [j.prefix for j in jobs], c.group_size,
                               c.n_kv_heads, num_m, include_self=include_self, subsets=subsets)
        emap, works, segs, merges = t["row_map"], t["works"], t["segs"], t["merges"]
        self.kv_tokens = t["kv_tokens"]
        self.n_works, self.n_segs, self.n_merge = len(works), len(segs), len(merges)
        dev = dm.device
        self.row_map = ops.to_device(emap.view(ops.ROWMAP_DTYPE).reshape(-1), dev)
        self.works = ops.to_device(works, dev)
        self.segs = ops.to_device(_per_layer_segs(segs, c.n_layers), dev)
        self.merges = ops.to_device(merges, dev) if len(merges) else None
        self.max_rows = t["max_rows"]
        self.rope = dm.rope_for(max(nt.max_pos, int(emap[:, 1].max())) + 1)
        self.part_rows = t["part_rows"]
        self._hd, self._part = hd, None
        self.n_real_works, self.n_real_segs = self.n_works, self.n_segs

    def _partials(self):
        # bf16 partials: a normalised partial row is a convex combination of V rows,
        # so one bf16 rounding (2^-9 relative) before the merge adds at most the
        # error of the final bf16 output; it halves the partial traffic.  Allocated
        # on first use: a plan that only feeds a captured graph never needs its own.
        if self._part is None:
            torch = _torch()
            n = max(self.part_rows, 1)
            dev = self.works.device
            self._part = (torch.empty((n, self._hd), dtype=torch.bfloat16, device=dev),
                          torch.empty((n,), dtype=torch.float32, device=dev))
        return self._part

    @property
    def part_o(self):
        return self._partials()[0]

    @part_o.setter
    def part_o(self, v):
        self._part = (v, self._partials()[1])

    @property
    def part_lse(self):
        return self._partials()[1]

    def pad_to(self, works_cap: int, segs_cap: int, rows_cap: int = 0, part_cap: int = 0) -> None:
        """Grow the device tables to fixed capacities (a captured graph's launch
        shape): extra works are empty (no segment, no row) and cost a CTA a
        few barrier round trips; extra segments are never referenced.
        rows_cap / part_cap: row-map entries and partial rows (a C5 shard's
        share of a batch varies with how the selections fall on it)."""
        torch = _torch()
        nb = rows_cap * ops.ROWMAP_DTYPE.itemsize  # the row map is a byte tensor
        if nb > self.row_map.numel():
            rm = torch.zeros(nb, dtype=torch.uint8, device=self.row_map.device)
            rm[: self.row_map.numel()].copy_(self.row_map)
            self.row_map = rm
        if part_cap > self.part_rows:
            self.part_rows = part_cap
            self._part = None
        L = self.segs.numel() // (self.n_segs * ops.SEG_DTYPE.itemsize) if self.n_segs else 0
        if works_cap < self.n_real_works or segs_cap < self.n_real_segs:
            raise ValueError("capacity below the schedule's size")
        w = torch.zeros(works_cap * ops.WORK_DTYPE.itemsize, dtype=torch.uint8, device=self.works.device)
        w[: self.works.numel()].copy_(self.works)
        s = torch.zeros((L, segs_cap * ops.SEG_DTYPE.itemsize), dtype=torch.uint8, device=self.segs.device)
        s[:, : self.n_segs * ops.SEG_DTYPE.itemsize].copy_(self.segs.view(L, -1))
        self.works, self.segs = w, s.view(-1)
        self.n_works, self.n_segs = works_cap, segs_cap

    def copy_tables_from(self, other: "ChunkMajorSchedule") -> None:
        """Load another batch's tables into these (padded) buffers in place."""
        if other.n_real_works > self.n_works or other.n_real_segs > self.n_segs:
            raise ValueError("schedule exceeds the captured capacity")
        nw = other.n_real_works * ops.WORK_DTYPE.itemsize
        self.works[:nw].copy_(other.works[:nw], non_blocking=True)
        self.works[nw:].zero_()
        L = self.segs.numel() // (self.n_segs * ops.SEG_DTYPE.itemsize)
        ns = other.n_real_segs * ops.SEG_DTYPE.itemsize
        self.segs.view(L, -1)[:, :ns].copy_(other.segs.view(L, -1)[:, :ns], non_blocking=True)
        if other.part_rows > self.part_rows:
            raise ValueError("schedule's partials exceed the captured capacity")
        if other.row_map.numel() > self.row_map.numel():
            raise ValueError("row map exceeds the captured capacity")
        self.row_map[: other.row_map.numel()].copy_(other.row_map, non_blocking=True)
        self.merges.copy_(other.merges, non_blocking=True)

    def segs_ptr(self, layer: int) -> int:
        return self.segs.data_ptr() + layer * self.n_segs * ops.SEG_DTYPE.itemsize

    def launch(self, dm, nt: NewTokens, layer, qkv, out, pool, part_o=None, part_lse=None):
        c = dm.config
        qw, kw = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
        if self.n_works == 0:
            return
        ops.attention(q=qkv, q_tok_stride=qw + 2 * kw, tok_pos=nt.pos, tok_lo=nt.lo, rope=self.rope,
                      pool=pool, aux=nt.aux(), n_heads=c.n_heads, n_kv_heads=c.n_kv_heads, head_dim=c.head_dim,
                      works_dev=self.works, n_works=self.n_works, segs_dev=self.segs_ptr(layer), num_m=self.num_m,
                      out=out, out_tok_stride=qw, part_o=self.part_o if part_o is None else part_o,
                      part_lse=self.part_lse if part_lse is None else part_lse, row_map=self.row_map,
                      one_seg_partials=True)


def chunk_major_tables(tables, n_new, pos_host, aux_row0, prefixes, gs: int, hkv: int, num_m: int = 2,
                       include_self: bool = True, subsets=None) -> dict:
    """Host tables of a chunk-major K3 launch (ChunkMajorSchedule), vectorised
    numpy: the row map, works (chunk works kv-major then balanced row slices,
    then each query's SELF works), segments (one FULL per distinct chunk, one
    SELF per query slab) and the K3m merge groups.  include_self=False (a C5
    shard that is not the self rank): no SELF works, so a query's splits are
    its local chunks alone (possibly none: its merge then yields O = 0, LSE =
    -inf).

    subsets (per job, ascending local token indices): only those tokens' rows
    (the last layer of a scored forward needs the scored rows alone).  Their
    own-token (SELF) works then go through the row map too, and the merge
    groups write a COMPACT output: the kept tokens back to back in job order."""
    slab = (128 * num_m) // gs
    if slab < 1:
        raise ConfigError(f"group size {gs} exceeds the {128 * num_m} rows of one K3 work")
    n_jobs = len(n_new)
    pos = np.asarray(pos_host, np.int64)
    n_new = np.asarray(n_new, np.int64)
    tok0 = np.concatenate([[0], np.cumsum(n_new)[:-1]]).astype(np.int64)
    if subsets is None:
        ns = n_new
        sub_cat = np.concatenate([np.arange(n, dtype=np.int64) for n in n_new]) if n_jobs else np.zeros(0, np.int64)
    else:
        subs = [np.asarray(x, np.int64) for x in subsets]
        ns = np.array([len(x) for x in subs], np.int64)
        sub_cat = np.concatenate(subs) if n_jobs else np.zeros(0, np.int64)
    sub_off = np.concatenate([[0], np.cumsum(ns)[:-1]]).astype(np.int64)  # job's first kept token (compact)
    tabs = [np.asarray(t, dtype=np.int64).reshape(-1, 3) for t in tables]
    n_ch = np.array([len(t) for t in tabs], np.int64)
    n_split = n_ch + int(include_self)
    tokbase = np.concatenate([[0], np.cumsum(n_split * ns)])
    kv_rows = int(tokbase[-1]) * gs  # partial rows per kv head
    # ---- (query, chunk) pairs grouped by chunk (pool row, length), queries ascending
    qi = np.repeat(np.arange(n_jobs), n_ch)
    ch = np.concatenate(tabs) if len(qi) else np.zeros((0, 3), np.int64)
    sidx = np.arange(len(qi)) - np.repeat(np.cumsum(n_ch) - n_ch, n_ch)
    order = np.lexsort((qi, ch[:, 1], ch[:, 0]))
    qi, ch, sidx = qi[order], ch[order], sidx[order]
    # ---- row-map entries: every (pair, kept token) in pair order
    ne = ns[qi]
    pair_e0 = np.cumsum(ne) - ne
    rep = np.repeat(np.arange(len(qi)), ne)
    local = np.arange(int(ne.sum())) - pair_e0[rep]
    q_rep = qi[rep]
    tok = tok0[q_rep] + sub_cat[sub_off[q_rep] + local]
    n_self_e = int(ns.sum()) if (subsets is not None and include_self) else 0
    emap = np.zeros((max(len(tok) + n_self_e, 1), 4), np.int32)
    if len(tok):
        emap[: len(tok), 0] = tok
        emap[: len(tok), 1] = pos[tok] - ch[rep, 2]
        emap[: len(tok), 2] = tokbase[q_rep] + sidx[rep] * ns[q_rep] + local
    # ---- one FULL segment + works per distinct chunk: kv-major, then balanced slices
    if len(qi):
        newkey = np.r_[True, (ch[1:, 0] != ch[:-1, 0]) | (ch[1:, 1] != ch[:-1, 1])]
        kstart = np.flatnonzero(newkey)
        e_cnt = np.add.reduceat(ne, kstart)
        e0 = pair_e0[kstart]
        k = -(-e_cnt // slab)
        size = -(-e_cnt // k)
        n_keys = len(kstart)
        blk = hkv * k  # works per chunk
        kw = np.repeat(np.arange(n_keys), blk)
        within = np.arange(int(blk.sum())) - np.repeat(np.cumsum(blk) - blk, blk)
        kv = within // k[kw]
        sl = within % k[kw]
        t0 = sl * size[kw]
        cw = np.zeros(len(kw), dtype=ops.WORK_DTYPE)
        cw["q_tok0"] = e0[kw] + t0
        cw["n_tok"] = np.minimum(size[kw], e_cnt[kw] - t0)
        cw["kv_head"] = kv
        cw["seg_begin"] = kw
        cw["seg_end"] = kw + 1
        cw["out_mode"] = nat.OUT_MAPPED
        cw["part_row0"] = kv.astype(np.int64) * kv_rows
        cseg = np.zeros(n_keys, dtype=ops.SEG_DTYPE)
        cseg["row0"] = ch[kstart, 0]
        cseg["n_tok"] = ch[kstart, 1]
        cseg["kind"] = SEG_FULL
    else:
        cw = np.zeros(0, dtype=ops.WORK_DTYPE)
        cseg = np.zeros(0, dtype=ops.SEG_DTYPE)
        n_keys = 0
    # ---- SELF works (each query's own tokens, causal tree) into its last split
    ks = -(-ns // slab) * int(include_self)
    ssize = -(-ns // np.maximum(ks, 1))
    sq = np.repeat(np.arange(n_jobs), ks)
    st0 = (np.arange(int(ks.sum())) - np.repeat(np.cumsum(ks) - ks, ks)) * ssize[sq]
    sn = np.minimum(ssize[sq], ns[sq] - st0)
    sseg = np.zeros(len(sq), dtype=ops.SEG_DTYPE)
    sseg["src"] = 1
    sseg["row0"] = np.asarray(aux_row0, np.int64)[sq]
    sseg["kind"] = SEG_SELF
    prefix = np.asarray(prefixes, np.int64)
    sw = np.zeros((len(sq), hkv), dtype=ops.WORK_DTYPE)
    kvs = np.arange(hkv)[None, :]
    sw["n_tok"] = sn[:, None]
    sw["self_tok0"] = tok0[sq][:, None]
    sw["kv_head"] = kvs
    sw["seg_begin"] = (n_keys + np.arange(len(sq)))[:, None]
    sw["seg_end"] = sw["seg_begin"] + 1
    sw["prefix"] = prefix[sq][:, None]
    if subsets is None:
        sseg["n_tok"] = st0 + sn  # the slab's keys: up to its last token
        sw["q_tok0"] = (tok0[sq] + st0)[:, None]
        sw["out_mode"] = nat.OUT_PARTIAL
        sw["part_row0"] = kvs * kv_rows + ((tokbase[sq] + n_ch[sq] * ns[sq] + st0) * gs)[:, None]
    elif n_self_e:
        # kept tokens' own rows through the row map (entries after the chunk pairs')
        e_self0 = len(tok) + sub_off  # first SELF entry of each job
        sj = np.repeat(np.arange(n_jobs), ns)
        sl_local = np.arange(n_self_e) - sub_off[sj]
        stok = tok0[sj] + sub_cat
        emap[len(tok): len(tok) + n_self_e, 0] = stok
        emap[len(tok): len(tok) + n_self_e, 1] = pos[stok]
        emap[len(tok): len(tok) + n_self_e, 2] = tokbase[sj] + n_ch[sj] * ns[sj] + sl_local
        last_local = sub_cat[sub_off[sq] + st0 + sn - 1]
        sseg["n_tok"] = last_local + 1  # keys up to the slab's last kept token
        sw["q_tok0"] = (e_self0[sq] + st0)[:, None]
        sw["out_mode"] = nat.OUT_MAPPED
        sw["part_row0"] = kvs * kv_rows
    works = np.concatenate([cw, sw.reshape(-1)])
    segs = np.concatenate([cseg, sseg])
    mg = np.zeros((n_jobs, hkv), dtype=ops.MERGE_DTYPE)
    mg["part_row0"] = kvs * kv_rows + (tokbase[:-1] * gs)[:, None]
    mg["rows"] = (ns * gs)[:, None]
    mg["n_splits"] = n_split[:, None]
    mg["q_tok0"] = (tok0 if subsets is None else sub_off)[:, None]
    mg["kv_head"] = kvs
    merges = mg.reshape(-1)
    return {"row_map": emap, "works": works, "segs": segs, "merges": merges,
            "kv_tokens": int(ch[:, 1].sum()) if len(qi) else 0,
            "max_rows": int((ns * gs).max()) if n_jobs else 0, "part_rows": kv_rows * hkv}


def stage2_schedule_kind(n_jobs: int) -> str:
    """'chunk' (chunk-major, rows of many queries per work) for batches, 'query'
    (split-KV per query) for a single query or when DBSA_STAGE2_SCHEDULE forces it."""
    import os

    forced = os.environ.get("DBSA_STAGE2_SCHEDULE")
    if forced in ("chunk", "query"):
        return forced
    return "chunk" if n_jobs >= 8 else "query"


def scored_local_rows(jobs):
    """Per label job, the ascending local indices of its scored rows (the rows
    LabelScorer keeps: the last query token and every fed label token,
    model.py:441-443 via label_job), i.e. the rows the last layer must produce."""
    out = []
    for j in jobs:
        rows = {j.prefix - 1}
        off = j.prefix
        for lab in j.labels:
            rows.update(range(off, off + len(lab) - 1))
            off += len(lab) - 1
        out.append(np.array(sorted(rows), np.int64))
    return out


def _last_layer_subset_enabled() -> bool:
    import os

    return os.environ.get("DBSA_LAST_SUBSET", "1") != "0"


class Stage2Plan:
    """Single-device tables for a batch of QueryJobs: NewTokens + a K3
    schedule over the jobs' chunk tables (chunk-major for batches, split-KV
    per query otherwise; see stage2_schedule_kind).  A chunk-major plan of
    label jobs also holds `last`: the last layer's schedule over the scored
    rows alone (chunk_major_tables subsets), whose merge writes them compactly
    in LabelScorer.keep order; `last` is None otherwise."""

    def __init__(self, dm, jobs, target_ctas: int | None = None, order: str = "query", schedule: str | None = None):
        self.new = NewTokens(dm, jobs)
        self.schedule = schedule or stage2_schedule_kind(len(jobs))
        self.last = None
        if self.schedule == "chunk":
            self.sched = ChunkMajorSchedule(dm, jobs, self.new)
            if jobs and all(j.labels is not None for j in jobs) and _last_layer_subset_enabled():
                self.last = ChunkMajorSchedule(dm, jobs, self.new, subsets=scored_local_rows(jobs))
        else:
            self.sched = AttnSchedule(dm, jobs, self.new, target_ctas=target_ctas, order=order)
        for name in ("tok0", "n_tok", "num_m", "pos", "lo", "ids", "pages", "n_pages", "aux_rows"):
            setattr(self, name, getattr(self.new, name))
        for name in ("works", "n_works", "n_segs", "n_merge", "merges", "max_rows", "rope", "kv_tokens"):
            setattr(self, name, getattr(self.sched, name))

    @property
    def part_o(self):
        return self.sched.part_o

    @property
    def part_lse(self):
        return self.sched.part_lse

    @property
    def k_aux(self):
        return self.new.k_aux

    @property
    def v_aux(self):
        return self.new.v_aux

    def segs_ptr(self, layer: int) -> int:
        return self.sched.segs_ptr(layer)


def _split_bounds(counts: np.ndarray, n_split: int) -> list[int]:
    """Cut a chunk list into n_split contiguous runs of ~equal token count."""
    n = len(counts)
    if n == 0:
        return [0] * (n_split + 1)
    cum = np.cumsum(counts)
    total = cum[-1]
    b = [0]
    for s in range(1, n_split):
        k = int(np.searchsorted(cum, total * s / n_split))
        k = min(max(k + 1, b[-1] + 1), n - (n_split - s))
        b.append(k)
    b.append(n)
    return b


def _merge_array(merges) -> np.ndarray:
    a = np.zeros(len(merges), dtype=ops.MERGE_DTYPE)
    m = np.asarray(merges, dtype=np.int64)
    for i, name in enumerate(ops.MERGE_DTYPE.names):
        a[name] = m[:, i]
    return a


def run_jobs(dm, store, jobs, target_ctas=None, plan=None, keep=None):
    """Forward every job's new tokens; returns (plan, fp32 hidden [n_tok, d]), or
    only the rows `keep` (LabelScorer.keep) when given."""
    c = dm.config
    plan = plan or Stage2Plan(dm, jobs, target_ctas)
    nt, sched = plan.new, plan.sched
    qw, kw = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
    stride = qw + 2 * kw
    pool = store.planes() if store is not None and store.k is not None else nt.aux()

    def write_kv(layer, qkv):
        ops.kv_write(qkv[:, qw:], qkv[:, qw + kw:], stride, nt.pos, dm.rope, nt.pages, nt.n_pages, nt.k_aux,
                     nt.v_aux, nt.aux_rows, 1, 0, c.n_kv_heads, c.head_dim)

    def attend(layer, qkv, out):
        # last layer of a scored forward: the scored rows alone, compact in keep order
        compact = keep is not None and plan.last is not None and layer == c.n_layers - 1
        sc = plan.last if compact else sched
        sc.launch(dm, nt, layer, qkv, out, pool)
        if sc.n_merge:
            ops.lse_merge(sc.part_o, sc.part_lse, sc.merges, sc.n_merge, sc.max_rows, c.n_heads,
                          c.n_kv_heads, c.head_dim, out, qw)
        return compact

    h = _decoder(dm, nt.ids, attend, write_kv, keep_last=keep)
    return plan, h


def shard_chunk_table(cache, units, ranges, rank):
    """(row, n_tok, delta) of the units of one query owned by `rank`, with
    GLOBAL new positions (all units count toward the re-positioned context)."""
    from . import parallel

    rows, new_start = [], 0
    for b, s0, e0 in units:
        n = e0 - s0
        if parallel.owner_of(b, ranges) == rank:
            ent = cache.blocks[b]
            rows.append((ent.row0 + s0, n, new_start - (ent.pos_start + s0)))
        new_start += n
    return np.asarray(rows, dtype=np.int64).reshape(-1, 3), new_start


class ShardedPlan:
    """Tables of one C5 batch over the local shards of a
    group-sharded cache: every query's ordered units are split by owner with
    GLOBAL new positions kept (shard_chunk_table), each local rank gets a
    chunk-major K3 schedule over its own chunks (bf16 partials; only the self
    rank also covers the queries' own tokens), a per-rank K3m merge turns a
    rank's partials into one (O, LSE) per (token, head), and the final K3m
    merges the gathered per-rank results: the single softmax over the
    concatenated key set of kernels.py:52-56, split by owner."""

    def __init__(self, dm, caches, ranges, units_per_query, query_ids, labels, world, self_rank=0):
        c = dm.config
        self.ranks = list(caches)
        tables = {r: [] for r in caches}
        jobs = []
        for q, units in zip(query_ids, units_per_query):
            n_ctx = sum(e - s0 for _, s0, e in units)
            for r in caches:
                tab, _ = shard_chunk_table(caches[r], units, ranges, r)
                tables[r].append(tab)
            jobs.append(label_job(np.zeros((0, 3), np.int64), n_ctx, q, labels))
        self.jobs = jobs
        self.new = NewTokens(dm, jobs)
        self.tok0, self.n_tok, self.num_m = self.new.tok0, self.new.n_tok, self.new.num_m
        self.scheds = {r: ChunkMajorSchedule(dm, jobs, self.new, chunk_tables=tables[r],
                                             include_self=(r == self_rank)) for r in caches}
        self.kv_tokens = sum(sc.kv_tokens for sc in self.scheds.values())
        # final merge: one group per (query, kv head), one split per rank
        gs, hkv = c.group_size, c.n_kv_heads
        mg = np.zeros((len(jobs), hkv), dtype=ops.MERGE_DTYPE)
        mg["rows"] = (np.asarray(self.new.n_new, np.int64) * gs)[:, None]
        mg["n_splits"] = world
        mg["q_tok0"] = self.new.tok0[:-1, None]
        mg["kv_head"] = np.arange(hkv)[None, :]
        self.merges = ops.to_device(mg.reshape(-1), dm.device)
        self.n_merge = len(jobs) * hkv
        self.max_rows = int(mg["rows"].max())
        self.rope = dm.rope_for(max(sc.rope.shape[0] for sc in self.scheds.values()))


class ShardedStage2:
    """C5 stage 2 over a group-sharded cache.  Per layer: each local rank runs
    its chunk-major K3 and the per-rank K3m merge into (O bf16, LSE fp32) per
    (token, head); the per-rank results are all-gathered (NCCL all-gather over
    NVLink; LocalComm stacks logical shards) and the final K3m merges the
    `world` splits in token layout into the attention output."""

    def __init__(self, dm, caches, comm, ranges, units_per_query=None, query_ids=None, labels=None, self_rank=0,
                 plan=None):
        torch = _torch()
        c = dm.config
        self.dm, self.caches, self.comm, self.ranges = dm, caches, comm, ranges
        self.plan = plan or ShardedPlan(dm, caches, ranges, units_per_query, query_ids, labels, comm.world,
                                        self_rank)
        n_local = len(caches)
        n_tok = self.plan.new.n_tok
        self.canon_o = torch.zeros((n_local, n_tok, c.n_heads * c.head_dim), dtype=torch.bfloat16, device=dm.device)
        self.canon_lse = torch.zeros((n_local, n_tok, c.n_heads), dtype=torch.float32, device=dm.device)

    @property
    def jobs(self):
        return self.plan.jobs

    def run(self, keep=None):
        """Forward of the batch; returns the fp32 final hidden states (the rows
        `keep` only, when given)."""
        c = self.dm.config
        plan = self.plan
        nt = plan.new
        qw, kw = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
        stride = qw + 2 * kw
        ranks = plan.ranks
        n_tok = nt.n_tok

        def write_kv(layer, qkv):
            ops.kv_write(qkv[:, qw:], qkv[:, qw + kw:], stride, nt.pos, self.dm.rope, nt.pages, nt.n_pages,
                         nt.k_aux, nt.v_aux, nt.aux_rows, 1, 0, c.n_kv_heads, c.head_dim)

        def attend(layer, qkv, out):
            for i, r in enumerate(ranks):
                sc = plan.scheds[r]
                sc.launch(self.dm, nt, layer, qkv, out, self.caches[r].store.planes())
                ops.lse_merge(sc.part_o, sc.part_lse, sc.merges, sc.n_merge, sc.max_rows, c.n_heads,
                              c.n_kv_heads, c.head_dim, self.canon_o[i], qw, out_lse=self.canon_lse[i])
            if len(ranks) == self.comm.world:
                go, gl = self.canon_o, self.canon_lse  # every shard is local: already [world, ...]
            else:
                go = self.comm.all_gather([self.canon_o[0]])
                gl = self.comm.all_gather([self.canon_lse[0]])
            ops.lse_merge(go, gl, plan.merges, plan.n_merge, plan.max_rows, c.n_heads, c.n_kv_heads, c.head_dim,
                          out, qw, split_stride=n_tok * c.n_heads, tok_layout=True)

        return _decoder(self.dm, nt.ids, attend, write_kv, keep_last=keep)

    def forward(self):
        return self.run()

    def scores(self):
        scorer = LabelScorer(self.dm, self.plan.new, self.plan.jobs, len(self.plan.jobs[0].labels))
        h = self.run(keep=scorer.keep)
        return scorer(self.dm, h, subset=True)


class GraphedShardedStage2:
    """One C5 batch step -- the sharded forward (per layer: K3 per local rank,
    per-rank K3m, all-gather, final K3m) plus label scoring -- captured as one
    CUDA graph, NCCL all-gathers included.  A shard's chunk-major tables vary
    with how a batch's selections fall on it, so they are padded to
    capacities (`headroom` over the template) and every later batch copies
    its tables in and replays."""

    def __init__(self, dm, caches, comm, plan, n_labels, headroom: float = 1.5):
        torch = _torch()
        self.dm, self.plan = dm, plan
        for sc in plan.scheds.values():
            h = lambda n: int(n * headroom) + 64  # noqa: E731
            sc.pad_to(-(-h(sc.n_real_works) // 64) * 64, -(-h(sc.n_real_segs) // 16) * 16,
                      rows_cap=h(sc.row_map.numel() // ops.ROWMAP_DTYPE.itemsize), part_cap=h(sc.part_rows))
        self.runner = ShardedStage2(dm, caches, comm, None, plan=plan)
        self.scorer = LabelScorer(dm, plan.new, plan.jobs, n_labels).private_copy()
        self._run()  # warm-up: workspaces, cuBLAS handles, NCCL communicator, kernel attributes
        torch.cuda.current_stream(dm.device).synchronize()
        self.graph = torch.cuda.CUDAGraph()
        n0 = ops.LAUNCHES
        # a capture stream of its own and thread-local capture mode: other threads may keep
        # launching (Runner.infer from a thread pool) while this one captures
        with torch.cuda.graph(self.graph, stream=torch.cuda.Stream(dm.device), capture_error_mode="thread_local"):
            self.scores, self.best = self._run()
        self.launches = ops.LAUNCHES - n0

    def _run(self):
        h = self.runner.run(keep=self.scorer.keep)
        return self.scorer(self.dm, h, subset=True)

    def fits(self, plan) -> bool:
        t = self.plan
        if plan.new.n_tok != t.new.n_tok or tuple(plan.new.n_new) != tuple(t.new.n_new) or plan.rope is not t.rope:
            return False
        for r, sc in plan.scheds.items():
            c = t.scheds[r]
            if (sc.n_real_works > c.n_works or sc.n_real_segs > c.n_segs or sc.part_rows > c.part_rows
                    or sc.row_map.numel() > c.row_map.numel()):
                return False
        return True

    def replay(self, plan, scorer):
        """Copy `plan`'s tables into the captured buffers and replay."""
        if not self.fits(plan):
            raise ValueError("batch does not fit the captured sharded graph")
        t = self.plan
        if plan is not t:
            for dst, src in [(t.new.pos, plan.new.pos), (t.new.lo, plan.new.lo), (t.new.ids, plan.new.ids),
                             (t.new.pages, plan.new.pages), (t.merges, plan.merges),
                             (self.scorer.rows, scorer.rows), (self.scorer.targets, scorer.targets),
                             (self.scorer.owner, scorer.owner), (self.scorer.label_row0, scorer.label_row0),
                             (self.scorer.keep, scorer.keep), (self.scorer.rows_in_keep, scorer.rows_in_keep)]:
                dst.copy_(src, non_blocking=True)
            for r, sc in plan.scheds.items():
                t.scheds[r].copy_tables_from(sc)
        self.graph.replay()
        ops.LAUNCHES += self.launches
        return self.scores, self.best


class GraphedStage2:
    """A stage-2 batch forward + label scoring captured as one CUDA graph.

    Every step of the forward is a fixed launch sequence for a given table
    shape (number of jobs, new tokens per job, chunks per job): cuBLAS GEMMs
    plus the sm_100a kernels.  The graph is captured once on a template plan.
    Later batches with the same shape copy their work / segment / token tables
    into the template's device buffers and replay, with no per-launch host
    work.  This matters most at batch 1, where ~320 launches per forward would
    otherwise be host-bound.
    """

    def __init__(self, dm, store, jobs, plan, n_labels, capacity=None):
        """capacity: optional (works, segments) lower bound for a chunk-major
        template (e.g. the largest tables of a set of batches to replay)."""
        torch = _torch()
        self.dm, self.store, self.plan = dm, store, plan
        self.scorer = LabelScorer(dm, plan, jobs, n_labels).private_copy()
        self.key = plan_key(plan, self.scorer)
        if isinstance(plan.sched, ChunkMajorSchedule):
            # the chunk-major table sizes vary with how a batch's selections
            # overlap: capture at a padded capacity, replay any batch that fits
            sc = plan.sched
            if capacity is None:  # headroom for batches whose selections overlap less
                nw, ns = sc.n_real_works * 17 // 16 + 64, sc.n_real_segs * 17 // 16 + 16
            else:
                nw, ns = max(sc.n_real_works, capacity[0]), max(sc.n_real_segs, capacity[1])
            sc.pad_to(-(-nw // 64) * 64, -(-ns // 16) * 16)
            plan.works, plan.n_works, plan.segs, plan.n_segs = sc.works, sc.n_works, sc.segs, sc.n_segs
            if plan.last is not None:  # the last layer's scored-rows schedule, same headroom
                la = plan.last
                nw, ns = la.n_real_works * 17 // 16 + 64, la.n_real_segs * 17 // 16 + 16
                la.pad_to(-(-nw // 64) * 64, -(-ns // 16) * 16)
        else:
            # replay() copies later batches' tables into these buffers: they must not be
            # the shared split-KV template tensors (AttnSchedule._from_template)
            sc = plan.sched
            sc.works = sc.works.clone()
            sc.merges = sc.merges.clone() if sc.merges is not None else None
            sc.cta_works = sc.cta_works.clone() if sc.cta_works is not None else None
            plan.works, plan.merges = sc.works, sc.merges
        self._run()  # warm-up: workspace allocation, cuBLAS handles, kernel attributes
        torch.cuda.current_stream(dm.device).synchronize()
        self.graph = torch.cuda.CUDAGraph()
        n0 = ops.LAUNCHES
        # a capture stream of its own and thread-local capture mode: other threads may keep
        # launching (Runner.infer from a thread pool) while this one captures
        with torch.cuda.graph(self.graph, stream=torch.cuda.Stream(dm.device), capture_error_mode="thread_local"):
            self.scores, self.best = self._run()
        self.launches = ops.LAUNCHES - n0

    def _run(self):
        _, h = run_jobs(self.dm, self.store, None, plan=self.plan, keep=self.scorer.keep)
        return self.scorer(self.dm, h, subset=True)

    def replay(self, plan, scorer):
        """Copy `plan`'s tables into the captured buffers and replay."""
        if plan_key(plan, scorer) != self.key:
            raise ValueError("plan shape differs from the captured graph")
        t, n = self.plan, plan
        if n is not t:
            pairs = [(t.new.pos, n.new.pos), (t.new.lo, n.new.lo), (t.new.ids, n.new.ids), (t.new.pages, n.new.pages),
                     (self.scorer.rows, scorer.rows), (self.scorer.targets, scorer.targets),
                     (self.scorer.owner, scorer.owner), (self.scorer.label_row0, scorer.label_row0),
                     (self.scorer.keep, scorer.keep), (self.scorer.rows_in_keep, scorer.rows_in_keep)]
            if isinstance(t.sched, ChunkMajorSchedule):
                t.sched.copy_tables_from(n.sched)
                if t.last is not None:
                    t.last.copy_tables_from(n.last)
            else:
                pairs += [(t.sched.works, n.sched.works), (t.sched.segs, n.sched.segs)]
                if t.sched.cta_works is not None:
                    pairs.append((t.sched.cta_works, n.sched.cta_works))
                if t.sched.merges is not None:
                    pairs.append((t.sched.merges, n.sched.merges))
            for dst, src in pairs:
                dst.copy_(src, non_blocking=True)
        if n.sched.rope is not t.sched.rope:
            raise ValueError("rope table was re-allocated; recapture")
        self.graph.replay()
        ops.LAUNCHES += self.launches
        return self.scores, self.best


def plan_key(plan, scorer):
    """Launch shape of a stage-2 batch: plans with equal keys can replay one
    captured graph.  Chunk-major table sizes are capacity-checked at replay
    instead (GraphedStage2 pads them)."""
    sc = plan.sched
    if isinstance(sc, ChunkMajorSchedule):
        tables = ("chunk", sc.row_map.numel(), sc.num_m, plan.last.row_map.numel() if plan.last is not None else -1)
    else:
        tables = ("query", sc.n_works, sc.n_segs, sc.n_ctas, getattr(sc, "one_seg", False))
    return (plan.new.n_tok, tuple(plan.new.n_new), plan.new.n_pages, tables, sc.n_merge, sc.part_rows,
            int(scorer.rows.numel()), int(scorer.keep.numel()), scorer.n_out, plan.new.num_m)


def fits_graph(graph, plan) -> bool:
    """Whether `plan` can replay `graph`: its chunk-major tables fit the
    captured capacity, and the rope table it needs is the captured one (a
    plan reaching past the table grows it, DeviceModel.rope_for, and the graph
    must then be recaptured)."""
    sc, t = plan.sched, graph.plan.sched
    if sc.rope is not t.rope:
        return False
    if not isinstance(sc, ChunkMajorSchedule):
        return True
    last_fits = plan.last is None or (plan.last.n_real_works <= graph.plan.last.n_works
                                      and plan.last.n_real_segs <= graph.plan.last.n_segs)
    return sc.n_real_works <= t.n_works and sc.n_real_segs <= t.n_segs and last_fits


def _final_logits(dm, h_rows):
    torch = _torch()
    x = ops.rmsnorm(h_rows, dm.out_norm, dm.config.norm_eps)
    return torch.mm(x, dm.lm_head, out_dtype=torch.float32)


_SCORER_TLS = __import__("threading").local()


def _scorer_tables():
    d = getattr(_SCORER_TLS, "cache", None)
    if d is None:
        d = _SCORER_TLS.cache = __import__("collections").OrderedDict()
    return d


class LabelScorer:
    """Row gather + lm_head + log-softmax gather for a batch of label jobs
    (model.py:441-443, pipeline.py:376-382)."""

    def __init__(self, dm, plan, jobs, n_labels):
        # the tables depend on the jobs' shapes and labels only: a per-thread LRU
        # reuses their device copies across batches (Runner.infer's host path)
        key = (tuple(int(x) for x in plan.tok0[:len(jobs)]), tuple(int(j.prefix) for j in jobs),
               tuple(tuple(tuple(int(t) for t in lab) for lab in j.labels) for j in jobs), int(n_labels), str(dm.device))
        cache = _scorer_tables()
        hit = cache.get(key)
        if hit is not None:
            cache.move_to_end(key)
            (self.keep, self.rows_in_keep, self.rows, self.targets, self.owner, self.label_row0,
             self.n_out, self.n_labels) = hit
            return
        rows, targets, owner = [], [], []
        for qi, j in enumerate(jobs):
            base = int(plan.tok0[qi])
            nq = j.prefix
            off = nq
            for li, lab in enumerate(j.labels):
                # label token k is predicted by the last query row (k = 0) or by
                # the fed label token k-1 at local index off + k - 1
                prev = base + nq - 1
                for k, tok in enumerate(lab):
                    rows.append(prev)
                    targets.append(tok)
                    owner.append(qi * n_labels + li)
                    prev = base + off + k
                off += len(lab) - 1
        dev = dm.device
        # distinct scored rows (the last query row serves every label): the last
        # layer's O projection and FFN run on these alone (run_jobs keep=)
        keep = np.unique(np.asarray(rows, np.int64))
        self.keep = ops.h2d(keep, dev)
        self.rows_in_keep = ops.h2d(np.searchsorted(keep, np.asarray(rows, np.int64)).astype(np.int64), dev)
        self.rows = ops.h2d(np.asarray(rows, np.int64), dev)
        self.targets = ops.h2d(np.asarray(targets, np.int32), dev)
        self.owner = ops.h2d(np.asarray(owner, np.int64), dev)
        # rows of output o are contiguous (appended label by label): their bounds
        counts = np.bincount(np.asarray(owner, np.int64), minlength=len(jobs) * n_labels)
        self.label_row0 = ops.h2d(np.concatenate([[0], np.cumsum(counts)]).astype(np.int32), dev)
        self.n_out = len(jobs) * n_labels
        self.n_labels = n_labels
        cache[key] = (self.keep, self.rows_in_keep, self.rows, self.targets, self.owner, self.label_row0,
                      self.n_out, self.n_labels)
        while len(cache) > 64:
            cache.popitem(last=False)

    def private_copy(self):
        """A copy whose tables are its own (a captured graph's scorer: replay()
        writes later batches' tables into them, so they must not be the shared
        cached ones)."""
        c = object.__new__(LabelScorer)
        for name in ("keep", "rows_in_keep", "rows", "targets", "owner", "label_row0"):
            setattr(c, name, getattr(self, name).clone())
        c.n_out, c.n_labels = self.n_out, self.n_labels
        return c

    def __call__(self, dm, h, subset: bool = False):
        """h: all rows' final hidden states, or (subset) only the rows `keep`.
        K5 (ops.label_score) scores every (row, label token) pair straight from
        the final-normed distinct rows: no logits in HBM."""
        x = ops.rmsnorm(h if subset else h.index_select(0, self.keep), dm.out_norm, dm.config.norm_eps)
        lp = ops.label_score(x, dm.lm_head_t, self.rows_in_keep, self.targets)
        return ops.label_reduce(lp, self.label_row0, self.n_out // self.n_labels, self.n_labels)


def score_labels(dm, assembled, query_ids, labels):
    """Per-label scores (host float array) of one query against `assembled`."""
    store, chunks, n_ctx = _ctx_of(assembled)
    job = label_job(chunks, n_ctx, query_ids, labels)
    plan = Stage2Plan(dm, [job])
    scorer = LabelScorer(dm, plan, [job], len(labels))
    _, h = run_jobs(dm, store, [job], plan=plan, keep=scorer.keep)
    scores, _ = scorer(dm, h, subset=True)
    return scores[0].double().cpu().numpy()


def forward_query(dm, assembled, query_ids):
    store, chunks, n_ctx = _ctx_of(assembled)
    n = len(query_ids)
    job = QueryJob(chunks, n_ctx, list(query_ids), list(range(n)), [0] * n, n)
    _, h = run_jobs(dm, store, [job])
    return _final_logits(dm, h).cpu().numpy()


def _ctx_of(assembled):
    if assembled is None or assembled.total_tokens == 0:
        return None, np.zeros((0, 3), np.int64), 0
    return assembled.cache.store, assembled.chunks, assembled.total_tokens


def logits_host(dm, hidden):
    torch = _torch()
    h = torch.as_tensor(np.asarray(hidden, np.float32)).to(dm.device)
    return _final_logits(dm, h).cpu().numpy()


def forward_explicit_context(dm, tokens, context):
    """forward_encode with host context arrays: the context (already rotated at
    its positions) goes into an aux page set, the new tokens into another."""
    torch = _torch()
    c = dm.config
    n_ctx, t = len(context), len(tokens)
    store = PageStore(c, dm.device, n_ctx + t)
    dev = dm.device
    rows = store.reserve([n_ctx, t] if n_ctx else [t])
    hdp = store.hdp
    if n_ctx:
        # context K is already rotated: write it unrotated-by-table (position 0 row = identity)
        zero = torch.zeros(n_ctx, dtype=torch.int32, device=dev)
        pages = ops.to_device(_pages_for([(0, n_ctx, rows[0])]), dev)
        for layer, (k, v) in enumerate(context.layers):
            ks = torch.from_numpy(np.ascontiguousarray(k, np.float32)).to(dev).to(torch.bfloat16)
            vs = torch.from_numpy(np.ascontiguousarray(v, np.float32)).to(dev).to(torch.bfloat16)
            ops.kv_write(ks.reshape(n_ctx, -1), vs.reshape(n_ctx, -1), c.n_kv_heads * c.head_dim, zero, dm.rope,
                         pages, -(-n_ctx // PAGE), store.k, store.v, store.rows, c.n_layers, layer, c.n_kv_heads,
                         c.head_dim)
    del hdp
    self_row = rows[-1]
    qw, kw = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
    stride = qw + 2 * kw
    pos = torch.tensor(np.asarray(tokens.positions, np.int32), device=dev)
    pages = ops.to_device(_pages_for([(0, t, self_row)]), dev)
    gs = c.group_size
    num_m = m_tiles(t * gs)
    slab = (128 * num_m) // gs
    segs, works = [], []
    for t0 in range(0, t, slab):
        nt = min(slab, t - t0)
        sb = len(segs)
        if n_ctx:
            segs.append((0, 0, rows[0], n_ctx, SEG_FULL, 0))
        segs.append((0, 0, self_row, t0 + nt, SEG_SELF, 0))
        for kv in range(c.n_kv_heads):
            works.append((t0, nt, 0, kv, sb, len(segs), 0, 0, 0))
    wdev = ops.to_device(_work_array(works), dev)
    sdev = ops.to_device(_per_layer_segs(_seg_array(segs), c.n_layers), dev)
    pre = []

    def write_kv(layer, qkv):
        ops.kv_write(qkv[:, qw:], qkv[:, qw + kw:], stride, pos, dm.rope, pages, -(-t // PAGE), store.k, store.v,
                     store.rows, c.n_layers, layer, c.n_kv_heads, c.head_dim)
        pre.append((qkv[:, qw:qw + kw].float().reshape(t, c.n_kv_heads, c.head_dim).cpu().numpy(),
                    qkv[:, qw + kw:].float().reshape(t, c.n_kv_heads, c.head_dim).cpu().numpy()))

    def attend(layer, qkv, out):
        ops.attention(q=qkv, q_tok_stride=stride, tok_pos=pos, tok_lo=None, rope=dm.rope,
                      pool=store.planes(), aux=None, n_heads=c.n_heads, n_kv_heads=c.n_kv_heads, head_dim=c.head_dim,
                      works_dev=wdev, n_works=len(works),
                      segs_dev=sdev.data_ptr() + layer * len(segs) * ops.SEG_DTYPE.itemsize, num_m=num_m, out=out,
                      out_tok_stride=qw)

    ids = torch.tensor(np.asarray(tokens.ids, np.int64), device=dev)
    h = _decoder(dm, ids, attend, write_kv)
    return pre, h.cpu().numpy()
