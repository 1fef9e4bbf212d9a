"""Kernel-level parity of the sm_100a kernels against float64 restatements of
the reference math (kernels.masked_attention kernels.py:73-100, rope
model.py:205-239, select/order retrieval.py:352-388).  Inputs are rounded to
bf16 first so the comparison isolates the kernel's own arithmetic.

Tolerances: attention outputs max-abs 2e-2 (bf16 P and output rounding, O(1)
magnitudes); top-k ids bit-exact.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2503_08640_b200 import ops  # noqa: E402


def _rope64(x, pos, theta):
    # x [T, H, hd] float64; paired halves (model.py:222-239)
    hd = x.shape[-1]
    f = ops.inv_freq(hd, theta)
    ang = np.asarray(pos, dtype=np.float64)[:, None] * f[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    lo, hi = x[..., : hd // 2], x[..., hd // 2:]
    return np.concatenate([lo * c - hi * s, lo * s + hi * c], axis=-1)


def _attend64(q, k, v, mask, scale):
    s = (q @ k.T) * scale
    s = np.where(mask, s, -np.inf)
    m = s.max(axis=1, keepdims=True)
    e = np.where(mask, np.exp(s - m), 0.0)
    return (e / e.sum(axis=1, keepdims=True)) @ v


class Pool:
    """Minimal page pool for kernel tests: groups of tokens written with K2w."""

    def __init__(self, n_kv, hd, lengths, layers=1, seed=0, theta=10000.0, dev="cuda"):
        g = torch.Generator().manual_seed(seed)
        self.n_kv, self.hd, self.hdp, self.theta = n_kv, hd, ops.hd_pad(hd), theta
        self.lengths = list(lengths)
        self.pos_start = np.concatenate([[0], np.cumsum(self.lengths)[:-1]]).astype(np.int64)
        self.page0 = []
        p = 0
        for n in self.lengths:
            self.page0.append(p)
            p += -(-n // ops.PAGE)
        self.rows = p * ops.PAGE
        T = sum(self.lengths)
        self.k_pre = torch.randn(layers, T, n_kv, hd, generator=g).to(torch.bfloat16)
        self.v = torch.randn(layers, T, n_kv, hd, generator=g).to(torch.bfloat16)
        self.kp = torch.zeros(layers, n_kv, self.rows, self.hdp, dtype=torch.bfloat16, device=dev)
        self.vp = torch.zeros(layers, n_kv, self.hdp, self.rows, dtype=torch.bfloat16, device=dev)
        self.rope = ops.rope_table(T + 4096, hd, theta, dev)
        pages = []
        for b, n in enumerate(self.lengths):
            for i in range(0, n, ops.PAGE):
                pages.append((int(self.pos_start[b]) + i, min(ops.PAGE, n - i), (self.page0[b] * ops.PAGE) + i, 0))
        pages = np.array(pages, dtype=np.int32).view(ops.PAGE_DTYPE).reshape(-1)
        pd = ops.to_device(pages, dev)
        pos = torch.arange(T, dtype=torch.int32, device=dev)
        for layer in range(layers):
            ks = self.k_pre[layer].to(dev).reshape(T, n_kv * hd)
            vs = self.v[layer].to(dev).reshape(T, n_kv * hd)
            ops.kv_write(ks, vs, n_kv * hd, pos, self.rope, pd, len(pages), self.kp, self.vp, self.rows,
                         layers, layer, n_kv, hd)
        torch.cuda.synchronize()

    def row0(self, b, start=0):
        return self.page0[b] * ops.PAGE + start

    def k_rot64(self, layer, b):
        s, n = int(self.pos_start[b]), self.lengths[b]
        k = self.k_pre[layer, s:s + n].double().numpy()
        return _rope64(k, np.arange(s, s + n), self.theta)

    def v64(self, layer, b):
        s, n = int(self.pos_start[b]), self.lengths[b]
        return self.v[layer, s:s + n].double().numpy()


@pytest.mark.parametrize("hd,theta", [(128, 500000.0), (64, 10000.0)])
def test_rope_tables_vs_float64(hd, theta):
    """dbsa_rope_table (float32) and dbsa_rope_table_f16 against (cos, sin) of
    pos * inv_freq in float64 (model.rope_angles, model.py:205-209): one
    rounding each, at positions up to 2^19."""
    rows = 1 << 19
    t = ops.rope_table(rows, hd, theta, "cuda")
    ang = np.arange(rows, dtype=np.float64)[:, None] * ops.inv_freq(hd, theta)[None, :]
    want = np.stack([np.cos(ang), np.sin(ang)], axis=-1)
    got32 = t.cpu().double().numpy()
    got16 = t.f16.cpu().double().numpy()
    assert np.abs(got32 - want).max() <= 2.0 ** -24
    assert np.abs(got16 - want).max() <= 2.0 ** -12


@pytest.mark.parametrize("hd,H,Hkv", [(128, 8, 2), (64, 4, 4), (16, 4, 2), (32, 2, 1), (8, 4, 2)])
def test_kv_write_pages(hd, H, Hkv):
    pool = Pool(Hkv, hd, [70, 64, 5, 130], layers=2, seed=1)
    for layer in range(2):
        for b in range(4):
            n, r0 = pool.lengths[b], pool.row0(b)
            got_k = pool.kp[layer, :, r0:r0 + n, :hd].float().cpu().numpy().transpose(1, 0, 2)
            want_k = pool.k_rot64(layer, b)
            assert np.abs(got_k - want_k).max() < 3e-2 * max(1.0, np.abs(want_k).max())
            got_v = pool.vp[layer, :, :hd, r0:r0 + n].float().cpu().numpy().transpose(2, 0, 1)
            np.testing.assert_array_equal(got_v, pool.v64(layer, b).astype(np.float32))
            # page tail and head-dim padding are zero
            tail = -(-n // ops.PAGE) * ops.PAGE
            assert pool.kp[layer, :, r0 + n:r0 + tail].abs().sum().item() == 0
            assert pool.kp[layer, :, r0:r0 + n, hd:].abs().sum().item() == 0


def _stage1_case(hd, H, Hkv, lengths, j=2, layer=0, layers=1, num_m=None, rope_f16=True):
    """Encode every group against sink + prev-j + self (masks.py:80-99) in one launch."""
    dev = "cuda"
    gs = H // Hkv
    pool = Pool(Hkv, hd, lengths, layers=layers, seed=7)
    assert hasattr(pool.rope, "f16")  # ops.rope_table builds the fp16 query-rotation table too
    if not rope_f16:
        del pool.rope.f16  # the float32 table for the Q staging as well
    T = sum(lengths)
    g = torch.Generator().manual_seed(3)
    q = torch.randn(T, H, hd, generator=g).to(torch.bfloat16)
    num_m = num_m or (2 if gs * 16 > 128 else 1)
    slab_tok = (128 * num_m) // gs
    works, segs = [], []
    for b, n in enumerate(lengths):
        ctx = sorted({0} | set(range(max(0, b - j), b)) - {b}) if b > 0 else []
        for kv in range(Hkv):
            for t0 in range(0, n, slab_tok):
                nt = min(slab_tok, n - t0)
                sb = len(segs)
                for c in ctx:
                    segs.append((0, layer, pool.row0(c), lengths[c], ops.nat.SEG_FULL, 0, 0, 0))
                segs.append((0, layer, pool.row0(b), t0 + nt, ops.nat.SEG_SELF, 0, 0, 0))
                works.append((int(pool.pos_start[b]) + t0, nt, int(pool.pos_start[b]), kv, sb, len(segs), 0, 0, 0))
    W = np.array([w[:8] for w in works], dtype=np.int32)
    wa = np.zeros(len(works), dtype=ops.WORK_DTYPE)
    for i, name in enumerate(ops.WORK_DTYPE.names[:8]):
        wa[name] = W[:, i]
    sa = np.array(segs, dtype=np.int32).view(ops.SEG_DTYPE).reshape(-1)
    out = torch.zeros(T, H, hd, dtype=torch.bfloat16, device=dev)
    qd = q.to(dev)
    pos = torch.arange(T, dtype=torch.int32, device=dev)
    ops.attention(q=qd, q_tok_stride=H * hd, tok_pos=pos, tok_lo=None, rope=pool.rope,
                  pool=(pool.kp, pool.vp, pool.rows, layers), aux=None, n_heads=H, n_kv_heads=Hkv, head_dim=hd,
                  works_dev=ops.to_device(wa, dev), n_works=len(wa), segs_dev=ops.to_device(sa, dev), num_m=num_m,
                  out=out, out_tok_stride=H * hd)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    q64 = _rope64(q.double().numpy(), np.arange(T), pool.theta)
    scale = 1.0 / math.sqrt(hd)
    worst = 0.0
    for b, n in enumerate(lengths):
        ctx = sorted({0} | set(range(max(0, b - j), b)) - {b}) if b > 0 else []
        s = int(pool.pos_start[b])
        for kv in range(Hkv):
            ks = [pool.k_rot64(layer, c)[:, kv] for c in ctx] + [pool.k_rot64(layer, b)[:, kv]]
            vs = [pool.v64(layer, c)[:, kv] for c in ctx] + [pool.v64(layer, b)[:, kv]]
            K, V = np.concatenate(ks), np.concatenate(vs)
            nctx = K.shape[0] - n
            mask = np.zeros((n, K.shape[0]), dtype=bool)
            mask[:, :nctx] = True
            mask[:, nctx:] = np.tril(np.ones((n, n), dtype=bool))
            for h in range(gs):
                head = kv * gs + h
                want = _attend64(q64[s:s + n, head], K, V, mask, scale)
                worst = max(worst, float(np.abs(got[s:s + n, head] - want).max()))
    return worst


@pytest.mark.parametrize("num_m", [1, 2])
@pytest.mark.parametrize("hd,H,Hkv", [(128, 8, 2), (128, 4, 4), (64, 8, 2), (16, 4, 2), (32, 6, 3), (32, 6, 2), (8, 4, 2)])
def test_stage1_block_sparse_attention(hd, H, Hkv, num_m):
    """num_m 1: single-M-tile kernel (Q in TMEM); 2: two ping-ponged M tiles."""
    worst = _stage1_case(hd, H, Hkv, [150, 64, 97, 200, 33], num_m=num_m)
    assert worst < 2e-2, worst


@pytest.mark.parametrize("hd,H,Hkv", [(128, 8, 2), (64, 8, 2)])
def test_stage1_attention_float32_query_rotation(hd, H, Hkv):
    """DbsaAttnArgs.rope_f16 = NULL: Q staging rotates with the float32 table."""
    assert _stage1_case(hd, H, Hkv, [150, 64, 97, 200, 33], num_m=2, rope_f16=False) < 2e-2


def test_stage1_attention_second_layer():
    assert _stage1_case(128, 8, 2, [65, 130, 64], layer=1, layers=2) < 2e-2


def _stage2_case(hd, H, Hkv, lengths, sel, n_q, labels, splits, theta=10000.0):
    """One query + label tree against selected (re-positioned) groups, with
    split-KV partials merged by K3m."""
    dev = "cuda"
    gs = H // Hkv
    pool = Pool(Hkv, hd, lengths, seed=11, theta=theta)
    Tp = sum(lengths[b] for b in sel)
    # new tokens: query (n_q) then each label (tree), positions Tp + index-in-branch
    n_new = n_q + sum(labels)
    pos = list(range(Tp, Tp + n_q))
    lo = [0] * n_q
    for L in labels:
        start = len(pos)
        pos += list(range(Tp + n_q, Tp + n_q + L))
        lo += [start] * L
    g = torch.Generator().manual_seed(5)
    qn = torch.randn(n_new, H, hd, generator=g).to(torch.bfloat16)
    kn = torch.randn(n_new, Hkv, hd, generator=g).to(torch.bfloat16)
    vn = torch.randn(n_new, Hkv, hd, generator=g).to(torch.bfloat16)
    aux_rows = -(-n_new // ops.PAGE) * ops.PAGE
    ka = torch.zeros(1, Hkv, aux_rows, pool.hdp, dtype=torch.bfloat16, device=dev)
    va = torch.zeros(1, Hkv, pool.hdp, aux_rows, dtype=torch.bfloat16, device=dev)
    posd = torch.tensor(pos, dtype=torch.int32, device=dev)
    pages = np.array([(i, min(ops.PAGE, n_new - i), i, 0) for i in range(0, n_new, ops.PAGE)],
                     dtype=np.int32).view(ops.PAGE_DTYPE).reshape(-1)
    ops.kv_write(kn.to(dev).reshape(n_new, -1), vn.to(dev).reshape(n_new, -1), Hkv * hd, posd, pool.rope,
                 ops.to_device(pages, dev), len(pages), ka, va, aux_rows, 1, 0, Hkv, hd)
    # chunks: selected groups at new positions; the queries of a chunk use rope
    # row (position - delta), delta = new_start - orig_start
    chunk_segs, new_start = [], 0
    for b in sel:
        chunk_segs.append((0, 0, pool.row0(b), lengths[b], ops.nat.SEG_FULL, new_start - int(pool.pos_start[b]), 0, 0))
        new_start += lengths[b]
    per = -(-len(chunk_segs) // splits)
    groups_segs = [chunk_segs[i:i + per] for i in range(0, len(chunk_segs), per)]
    groups_segs[-1] = groups_segs[-1] + [(1, 0, 0, n_new, ops.nat.SEG_SELF, 0, 0, 0)]
    S = len(groups_segs)
    num_m = 2 if n_new * gs > 128 else 1
    assert n_new * gs <= 128 * num_m
    rows = n_new * gs
    works, segs = [], []
    mgroups = []
    for kv in range(Hkv):
        base = kv * S * rows
        for s, gseg in enumerate(groups_segs):
            sb = len(segs)
            segs += gseg
            works.append((0, n_new, 0, kv, sb, len(segs), n_q, 1 if S > 1 else 0, base + s * rows))
        mgroups.append((base, rows, S, 0, kv))
    wa = np.zeros(len(works), dtype=ops.WORK_DTYPE)
    for i, name in enumerate(ops.WORK_DTYPE.names):
        wa[name] = [w[i] for w in works]
    sa = np.array(segs, dtype=np.int32).view(ops.SEG_DTYPE).reshape(-1)
    out = torch.zeros(n_new, H, hd, dtype=torch.bfloat16, device=dev)
    part_o = torch.zeros(Hkv * S * rows, hd, dtype=torch.float32, device=dev)
    part_l = torch.zeros(Hkv * S * rows, dtype=torch.float32, device=dev)
    ops.attention(q=qn.to(dev), q_tok_stride=H * hd, tok_pos=posd, tok_lo=torch.tensor(lo, dtype=torch.int32,
                  device=dev), rope=pool.rope, pool=(pool.kp, pool.vp, pool.rows, 1), aux=(ka, va, aux_rows, 1),
                  n_heads=H, n_kv_heads=Hkv, head_dim=hd, works_dev=ops.to_device(wa, dev), n_works=len(wa),
                  segs_dev=ops.to_device(sa, dev), num_m=num_m, out=out, out_tok_stride=H * hd, part_o=part_o,
                  part_lse=part_l)
    if S > 1:
        ma = np.zeros(len(mgroups), dtype=ops.MERGE_DTYPE)
        for i, name in enumerate(ops.MERGE_DTYPE.names):
            ma[name] = [m[i] for m in mgroups]
        ops.lse_merge(part_o, part_l, ops.to_device(ma, dev), len(ma), rows, H, Hkv, hd, out, H * hd)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    # reference: assemble (rotate K at new positions 0..Tp-1), query at own positions, tree mask
    Kc = np.concatenate([pool.k_pre[0, int(pool.pos_start[b]):int(pool.pos_start[b]) + lengths[b]].double().numpy()
                         for b in sel])
    Kc = _rope64(Kc, np.arange(Tp), theta)
    Vc = np.concatenate([pool.v64(0, b) for b in sel])
    Kn = _rope64(kn.double().numpy(), pos, theta)
    q64 = _rope64(qn.double().numpy(), pos, theta)
    K = np.concatenate([Kc, Kn])
    V = np.concatenate([Vc, vn.double().numpy()])
    mask = np.zeros((n_new, Tp + n_new), dtype=bool)
    mask[:, :Tp] = True
    for r in range(n_new):
        for k in range(n_new):
            mask[r, Tp + k] = k <= r and (k < n_q or k >= lo[r])
    worst = 0.0
    for kv in range(Hkv):
        for h in range(gs):
            head = kv * gs + h
            want = _attend64(q64[:, head], K[:, kv], V[:, kv], mask, 1.0 / math.sqrt(hd))
            worst = max(worst, float(np.abs(got[:, head] - want).max()))
    return worst


@pytest.mark.parametrize("splits", [1, 2, 3])
@pytest.mark.parametrize("hd,H,Hkv,theta", [(128, 8, 2, 500000.0), (16, 4, 2, 10000.0), (64, 4, 4, 10000.0)])
@pytest.mark.parametrize("n_q,labels", [(20, [4, 6, 3, 5]), (10, [3, 4, 2, 3])])
def test_stage2_split_kv_attention(hd, H, Hkv, theta, splits, n_q, labels):
    """(20, ...) runs the two-M-tile kernel at gs 4, (10, ...) the single-M-tile one."""
    worst = _stage2_case(hd, H, Hkv, [100, 64, 300, 77, 150, 90], sel=[0, 2, 3, 5], n_q=n_q, labels=labels,
                         splits=splits, theta=theta)
    assert worst < 2e-2, worst


def _py_select(scores, budget, ordering):
    n = len(scores)
    cand = sorted(range(1, n), key=lambda u: (-scores[u], u))[: budget - 1]
    if ordering == "in-order":
        cand.sort()
    elif ordering == "low-to-high":
        cand.sort(key=lambda u: (scores[u], u))
    else:
        cand.sort(key=lambda u: -u)
    return [0] + cand


@pytest.mark.parametrize("n_units", [1, 2, 16, 60, 997])
@pytest.mark.parametrize("ordering", ["in-order", "low-to-high", "reverse"])
def test_topk_bit_exact(n_units, ordering):
    rng = np.random.default_rng(n_units)
    scores = rng.random((33, n_units))
    scores[:, ::3] = np.round(scores[:, ::3], 1)  # ties
    scores[0] = 0.0                               # all tied
    dev_scores = torch.from_numpy(scores).cuda()
    for ratio in (0.1, 0.3, 0.5, 1.0):
        budget = math.ceil(ratio * n_units)
        got = ops.topk_select(dev_scores, budget, ordering).cpu().numpy()
        for q in range(scores.shape[0]):
            assert list(got[q]) == _py_select(list(scores[q]), budget, ordering)


@pytest.mark.parametrize("n_units", [257, 3001, 40000])
@pytest.mark.parametrize("ordering", ["in-order", "low-to-high", "reverse"])
def test_topk_radix_bit_exact(n_units, ordering):
    """K4 above 256 units (example granularity: thousands of demonstrations)
    runs the radix select; bit-exact with the reference's sort
    (retrieval.py:352-388) with ties, all-tied rows, +-0.0 and negative scores."""
    rng = np.random.default_rng(n_units)
    scores = rng.random((9, n_units)) * 20 - 5
    scores[:, ::3] = np.round(scores[:, ::3], 0)  # many ties
    scores[0] = 0.0                               # all tied
    scores[1, ::2] = -0.0                         # -0.0 ties +0.0 (Python compares them equal)
    dev_scores = torch.from_numpy(scores).cuda()
    for ratio in (0.001, 0.3, 1.0):
        budget = max(1, math.ceil(ratio * n_units))
        got = ops.topk_select(dev_scores, budget, ordering).cpu().numpy()
        for q in range(scores.shape[0]):
            assert list(got[q]) == _py_select(list(scores[q]), budget, ordering), (q, budget)


class _DM:
    """The attributes a stage-2 plan reads (config, device, rope tables)."""

    def __init__(self, cfg, dev):
        self.config, self.device = cfg, dev
        self.rope = ops.rope_table(cfg.max_seq_len, cfg.head_dim, cfg.rope_theta, dev)

    def rope_for(self, rows):
        if rows > self.rope.shape[0]:
            self.rope = ops.rope_table(rows, self.config.head_dim, self.config.rope_theta, self.device)
        return self.rope


@pytest.mark.parametrize("schedule", ["chunk", "query", "chunk-padded"])
@pytest.mark.parametrize("hd,H,Hkv", [(128, 8, 2), (64, 4, 4), (32, 8, 1), (128, 4, 4), (128, 16, 2), (64, 6, 2)])
def test_stage2_batch_schedules_vs_float64(schedule, hd, H, Hkv):
    """(128, 4, 4): MHA at head_dim 128 (C4's layout, 256-token chunk works);
    (128, 16, 2): GQA-8 (the 70B shape's grouping, 32-token works)."""
    """A batch of label jobs over overlapping chunk tables (whole groups and
    example-granularity sub-spans, assorted orders) through one layer of K3 +
    K3m, chunk-major (DBSA_OUT_MAPPED row-map works) and split-KV per query,
    against float64 attention over the assembled context (kvstore.py:188-221,
    model.py:381-392, kernels.py:73-100)."""
    import paper_2503_08640_b200 as P
    from paper_2503_08640_b200 import engine

    dev = torch.device("cuda", 0)
    theta = 10000.0
    cfg = P.ModelConfig(d_model=H * hd, n_layers=1, n_heads=H, n_kv_heads=Hkv, head_dim=hd, ffn_dim=64,
                        vocab_size=300, rope_theta=theta, max_seq_len=8192)
    dm = _DM(cfg, dev)
    lengths = [130, 64, 300, 77, 150, 90, 200, 41]
    cache = P.SegmentedKVCache(cfg, dev, capacity_tokens=sum(lengths))
    blocks = cache._reserve(lengths, [b"\0" * 32] * len(lengths), [()] * len(lengths))
    g = torch.Generator(device=dev).manual_seed(3)
    cache.store.k.normal_(generator=g)
    cache.store.v.normal_(generator=g)
    st = cache.store
    rows0 = np.array([b.row0 for b in blocks])
    pos0 = np.array([b.pos_start for b in blocks])
    rng = np.random.default_rng(7)
    # units: whole groups plus a few sub-spans (example granularity)
    units = [(b, 0, n) for b, n in enumerate(lengths)] + [(2, 10, 70), (2, 200, 300), (6, 5, 133), (4, 0, 64)]
    jobs = []
    for qi in range(11):
        k = int(rng.integers(1, 6))
        pick = [0] + rng.choice(np.arange(1, len(units)), k - 1, replace=False).tolist()
        if qi % 3 == 1:
            pick = [0] + pick[1:][::-1]
        ln = np.array([units[u][2] - units[u][1] for u in pick])
        new_start = np.cumsum(ln) - ln
        tab = np.array([(rows0[units[u][0]] + units[u][1], ln[i], new_start[i] - (pos0[units[u][0]] + units[u][1]))
                        for i, u in enumerate(pick)])
        q_ids = rng.integers(3, 200, int(rng.integers(5, 30))).tolist()
        labels = [rng.integers(3, 200, int(rng.integers(2, 6))).tolist() for _ in range(3)]
        jobs.append((engine.label_job(tab, int(ln.sum()), q_ids, labels), pick, ln))
    plan = engine.Stage2Plan(dm, [j for j, _, _ in jobs], schedule=schedule.split("-")[0])
    if schedule == "chunk-padded":  # graph capacity padding: trailing empty works / unused segments
        plan.sched.pad_to(plan.sched.n_works + 300, plan.sched.n_segs + 20)
    nt = plan.new
    qw, kw = H * hd, Hkv * hd
    qkv = (torch.randn(nt.n_tok, qw + 2 * kw, generator=g, device=dev) * 0.5).to(torch.bfloat16)
    ops.kv_write(qkv[:, qw:], qkv[:, qw + kw:], qw + 2 * kw, nt.pos, dm.rope, nt.pages, nt.n_pages, nt.k_aux,
                 nt.v_aux, nt.aux_rows, 1, 0, Hkv, hd)
    out = torch.zeros(nt.n_tok, qw, dtype=torch.bfloat16, device=dev)
    plan.sched.launch(dm, nt, 0, qkv, out, st.planes())
    if plan.sched.n_merge:
        ops.lse_merge(plan.sched.part_o, plan.sched.part_lse, plan.sched.merges, plan.sched.n_merge,
                      plan.sched.max_rows, H, Hkv, hd, out, qw)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy().reshape(nt.n_tok, H, hd)
    Kp = st.k[0].float().cpu().numpy()  # [Hkv][rows][hdp], rotated at original positions
    Vp = st.v[0].float().cpu().numpy()  # [Hkv][hdp][rows]
    qn = qkv[:, :qw].float().cpu().numpy().reshape(nt.n_tok, H, hd).astype(np.float64)
    kn = qkv[:, qw:qw + kw].float().cpu().numpy().reshape(nt.n_tok, Hkv, hd).astype(np.float64)
    vn = qkv[:, qw + kw:].float().cpu().numpy().reshape(nt.n_tok, Hkv, hd).astype(np.float64)
    gs = H // Hkv
    worst = 0.0
    for qi, (job, pick, ln) in enumerate(jobs):
        t0, n = int(nt.tok0[qi]), nt.n_new[qi]
        pos = nt.pos_host[t0:t0 + n].astype(np.int64)
        ch = np.asarray(job.chunks).reshape(-1, 3)
        for kv in range(Hkv):
            kself = _rope64(kn[t0:t0 + n, kv:kv + 1], pos, theta)[:, 0]
            for h in range(gs):
                head = kv * gs + h
                q = qn[t0:t0 + n, head:head + 1]
                scores, vals = [], []
                for row, cnt, delta in ch:
                    qr = _rope64(q, pos - delta, theta)[:, 0]  # R(p - delta) q . R(p_orig) k
                    scores.append(qr @ Kp[kv, row:row + cnt, :hd].astype(np.float64).T)
                    vals.append(Vp[kv, :hd, row:row + cnt].astype(np.float64).T)
                qs = _rope64(q, pos, theta)[:, 0]
                s_self = qs @ kself.T
                lo = np.asarray(job.lo)
                vis = np.zeros((n, n), bool)
                for r in range(n):
                    for kk in range(r + 1):
                        vis[r, kk] = kk < job.prefix or kk >= lo[r]
                s_self = np.where(vis, s_self, -np.inf)
                s = np.concatenate(scores + [s_self], axis=1) / math.sqrt(hd)
                v = np.concatenate(vals + [vn[t0:t0 + n, kv]], axis=0)
                m = s.max(axis=1, keepdims=True)
                e = np.exp(s - m)
                want = (e / e.sum(axis=1, keepdims=True)) @ v
                worst = max(worst, float(np.abs(got[t0:t0 + n, head] - want).max()))
    assert worst < 2e-2, worst


@pytest.mark.parametrize("n_splits", [1, 7, 19, 40, 70])
@pytest.mark.parametrize("dtype", ["bf16", "bf16-chunked", "fp32"])
def test_lse_merge_large_vs_torch(n_splits, dtype):
    """K3m on a merge large enough for the throughput kernels (the chunk-major
    batch shape: many groups of 176 rows, bf16 or fp32 partials, some splits
    empty): the single softmax over the concatenated key set (kernels.py:52-56)
    recomputed in float64 from the same partials.  bf16-chunked: the partials
    in the 16-column chunk layout (DbsaMergeArgs.part_chunk_rows) K3 writes."""
    dev = torch.device("cuda", 0)
    H, Hkv, hd = 32, 8, 128
    gs = H // Hkv
    n_q, n_tok = 24, 44
    rows = n_tok * gs
    g = torch.Generator(device=dev).manual_seed(n_splits)
    part_dtype = torch.float32 if dtype == "fp32" else torch.bfloat16
    n_groups = n_q * Hkv
    part_o = torch.randn(n_groups * n_splits * rows, hd, generator=g, device=dev).to(part_dtype)
    part_lse = torch.randn(n_groups * n_splits * rows, generator=g, device=dev) * 3
    part_lse[torch.rand(part_lse.shape, generator=g, device=dev) < 0.05] = -float("inf")  # empty splits
    groups = np.zeros(n_groups, dtype=ops.MERGE_DTYPE)
    for q in range(n_q):
        for kv in range(Hkv):
            i = q * Hkv + kv
            groups[i] = (i * n_splits * rows, rows, n_splits, q * n_tok, kv)
    out = torch.zeros(n_q * n_tok, H * hd, dtype=torch.bfloat16, device=dev)
    if dtype == "bf16-chunked":
        R = part_o.shape[0]
        chunked = part_o.view(R, hd // 16, 16).transpose(0, 1).contiguous().view(R, hd)  # [hd/16][R][16] in memory
        ops.lse_merge(chunked, part_lse, ops.to_device(groups, dev), n_groups, rows, H, Hkv, hd, out, H * hd,
                      part_chunk_rows=R)
    else:
        ops.lse_merge(part_o, part_lse, ops.to_device(groups, dev), n_groups, rows, H, Hkv, hd, out, H * hd,
                      part_chunk_rows=0)
    torch.cuda.synchronize()
    po = part_o.double().view(n_groups, n_splits, rows, hd)
    pl = part_lse.double().view(n_groups, n_splits, rows)
    lse = torch.logsumexp(pl, dim=1, keepdim=True)
    w = torch.nan_to_num(torch.exp(pl - lse), nan=0.0)
    want = (w.unsqueeze(-1) * po).sum(1)  # [n_groups, rows, hd]
    want = want.view(n_q, Hkv, n_tok, gs, hd).permute(0, 2, 1, 3, 4).reshape(n_q * n_tok, H * hd)
    err = float((out.double() - want).abs().max())
    assert err < 2e-2, err


@pytest.mark.parametrize("n_local", [1, 24])
@pytest.mark.parametrize("chunked", [False, True])
def test_lse_merge_two_level_equals_one_level(n_local, chunked):
    """The C5 merge (engine.ShardedStage2): each of 3 "ranks" merges its own
    splits into a bf16 (O, LSE) per (token, head) (out_lse mode; a rank with
    no split for a row yields O = 0, LSE = -inf), and the token-layout merge
    of the 3 results equals the single softmax over all splits
    (kernels.py:52-56) within the bf16 tolerance.  chunked: the per-rank
    partials in K3's 16-column chunk layout (the chunk-major schedule's), which
    at 12 queries takes the wide K3m form in out_lse mode."""
    dev = torch.device("cuda", 0)
    H, Hkv, hd = 32, 8, 128
    gs = H // Hkv
    n_q, n_tok = (4 if n_local == 1 else 12), 44  # 12 queries: the throughput kernel path
    rows = n_tok * gs
    world = 3
    g = torch.Generator(device=dev).manual_seed(n_local)
    n_groups = n_q * Hkv
    T = n_q * n_tok
    splits = [n_local, 0 if n_local > 1 else 1, n_local]  # rank 1 holds nothing for these queries (n_local > 1)
    parts = []
    canon_o = torch.zeros(world, T, H * hd, dtype=torch.bfloat16, device=dev)
    canon_lse = torch.zeros(world, T, H, dtype=torch.float32, device=dev)
    for r in range(world):
        ns = splits[r]
        po = torch.randn(max(1, n_groups * ns * rows), hd, generator=g, device=dev).to(torch.bfloat16)
        pl = torch.randn(max(1, n_groups * ns * rows), generator=g, device=dev) * 3
        grp = np.zeros(n_groups, dtype=ops.MERGE_DTYPE)
        for q in range(n_q):
            for kv in range(Hkv):
                i = q * Hkv + kv
                grp[i] = (i * ns * rows, rows, ns, q * n_tok, kv)
        if chunked:
            R = po.shape[0]
            po_c = po.view(R, hd // 16, 16).transpose(0, 1).contiguous().view(R, hd)
            ops.lse_merge(po_c, pl, ops.to_device(grp, dev), n_groups, rows, H, Hkv, hd, canon_o[r], H * hd,
                          out_lse=canon_lse[r], part_chunk_rows=R)
        else:
            ops.lse_merge(po, pl, ops.to_device(grp, dev), n_groups, rows, H, Hkv, hd, canon_o[r], H * hd,
                          out_lse=canon_lse[r], part_chunk_rows=0)
        parts.append((po[: n_groups * ns * rows].double().view(n_groups, ns, rows, hd),
                      pl[: n_groups * ns * rows].double().view(n_groups, ns, rows)))
    fin = np.zeros(n_groups, dtype=ops.MERGE_DTYPE)
    for q in range(n_q):
        for kv in range(Hkv):
            fin[q * Hkv + kv] = (0, rows, world, q * n_tok, kv)
    out = torch.zeros(T, H * hd, dtype=torch.bfloat16, device=dev)
    ops.lse_merge(canon_o, canon_lse, ops.to_device(fin, dev), n_groups, rows, H, Hkv, hd, out, H * hd,
                  split_stride=T * H, tok_layout=True)
    torch.cuda.synchronize()
    po = torch.cat([p[0] for p in parts], dim=1)
    pl = torch.cat([p[1] for p in parts], dim=1)
    lse = torch.logsumexp(pl, dim=1, keepdim=True)
    w = torch.exp(pl - lse)
    want = (w.unsqueeze(-1) * po).sum(1).view(n_q, Hkv, n_tok, gs, hd).permute(0, 2, 1, 3, 4).reshape(T, H * hd)
    err = float((out.double() - want).abs().max())
    # two bf16 roundings (the per-rank O, the output) of N(0, 1) partial values:
    # 2 x 2^-9 relative each, with a 2x margin
    tol = 4 * 2.0 ** -9 * float(want.abs().max()) + 1e-3
    assert err < tol, (err, tol)
    if n_local > 1:  # the empty rank's rows: O = 0, LSE = -inf
        assert torch.all(canon_lse[1] == -float("inf")) and torch.all(canon_o[1] == 0)
    # per-rank LSE = logsumexp of that rank's splits, token-major
    l0 = torch.logsumexp(parts[0][1], dim=1).view(n_q, Hkv, n_tok, gs).permute(0, 2, 1, 3).reshape(T, H)
    assert float((canon_lse[0].double() - l0).abs().max()) < 1e-4


# ---------------------------------------------------------------- north-star shapes
def _rope64_t(x, pos, theta):
    """torch float64 paired-halves RoPE (model.py:222-239); x [..., T, hd], pos [T]."""
    hd = x.shape[-1]
    f = torch.from_numpy(ops.inv_freq(hd, theta)).to(x.device)
    ang = pos.double()[:, None] * f[None, :]
    c, s = torch.cos(ang), torch.sin(ang)
    lo, hi = x[..., : hd // 2], x[..., hd // 2:]
    return torch.cat([lo * c - hi * s, lo * s + hi * c], dim=-1)


def _stage2_at_scale(H, Hkv, hd, theta, n_groups, group_tok, budget, n_queries, q_tok, labels, check, seed=0,
                     mode="chunk"):
    """One layer of K3 + K3m at a north-star shape against float64 attention
    over the ASSEMBLED context: selected groups' keys rotated at their new
    positions 0..T'-1 (kvstore.assemble, kvstore.py:188-221), queries at their
    own positions T'+i, the query/label tree mask (model.py:381-392), softmax
    in float64 (kernels.py:43-100).  mode: "chunk" (chunk-major, bf16
    partials), "chunk-last" (the last layer's schedule over the scored rows
    only: mapped SELF works, compact output), "query" (split-KV as Runner.infer
    runs it: cost-packed CTA ranges, SELF as its own split, bf16 partials)."""
    import paper_2503_08640_b200 as P
    from paper_2503_08640_b200 import engine

    dev = torch.device("cuda", 0)
    cfg = P.ModelConfig(d_model=H * hd, n_layers=1, n_heads=H, n_kv_heads=Hkv, head_dim=hd, ffn_dim=64,
                        vocab_size=300, rope_theta=theta, max_seq_len=131072)
    dm = _DM(cfg, dev)
    cache = P.SegmentedKVCache(cfg, dev, capacity_tokens=n_groups * group_tok)
    blocks = cache._reserve([group_tok] * n_groups, [b"\0" * 32] * n_groups, [()] * n_groups)
    g = torch.Generator(device=dev).manual_seed(seed)
    st = cache.store
    st.k.normal_(generator=g)
    st.v.normal_(generator=g)
    for e in blocks:  # page tails stay zero, as K2w leaves them
        tail = -(-e.token_count // ops.PAGE) * ops.PAGE
        st.k[:, :, e.row0 + e.token_count:e.row0 + tail] = 0
        st.v[..., e.row0 + e.token_count:e.row0 + tail] = 0
    rng = np.random.default_rng(seed)
    rows0 = np.array([e.row0 for e in blocks])
    pos0 = np.array([e.pos_start for e in blocks])
    jobs, picks = [], []
    for qi in range(n_queries):
        pick = np.concatenate([[0], np.sort(rng.choice(np.arange(1, n_groups), budget - 1, replace=False))])
        ln = np.full(budget, group_tok)
        new_start = np.cumsum(ln) - ln
        tab = np.stack([rows0[pick], ln, new_start - pos0[pick]], axis=1)
        q_ids = rng.integers(3, 200, q_tok).tolist()
        labs = [rng.integers(3, 200, labels[1]).tolist() for _ in range(labels[0])]
        jobs.append(engine.label_job(tab, int(ln.sum()), q_ids, labs))
        picks.append(pick)
    plan = engine.Stage2Plan(dm, jobs, schedule="query" if mode == "query" else "chunk")
    sched = plan.last if mode == "chunk-last" else plan.sched
    assert sched is not None and sched.part_o.dtype == torch.bfloat16
    if mode == "query":
        assert sched.cta_works is not None
    nt = plan.new
    qw, kw = H * hd, Hkv * hd
    qkv = (torch.randn(nt.n_tok, qw + 2 * kw, generator=g, device=dev) * 0.5).to(torch.bfloat16)
    ops.kv_write(qkv[:, qw:], qkv[:, qw + kw:], qw + 2 * kw, nt.pos, dm.rope, nt.pages, nt.n_pages, nt.k_aux,
                 nt.v_aux, nt.aux_rows, 1, 0, Hkv, hd)
    out = torch.zeros(nt.n_tok, qw, dtype=torch.bfloat16, device=dev)
    sched.launch(dm, nt, 0, qkv, out, st.planes())
    ops.lse_merge(sched.part_o, sched.part_lse, sched.merges, sched.n_merge, sched.max_rows, H, Hkv, hd, out, qw)
    torch.cuda.synchronize()
    kept = engine.scored_local_rows(jobs)
    koff = np.concatenate([[0], np.cumsum([len(x) for x in kept])])
    gs = H // Hkv
    scale = 1.0 / math.sqrt(hd)
    worst = 0.0
    for qi in check:
        job, pick = jobs[qi], picks[qi]
        t0, n = int(nt.tok0[qi]), nt.n_new[qi]
        Tp = budget * group_tok
        pos = torch.from_numpy(nt.pos_host[t0:t0 + n].astype(np.int64)).to(dev)
        # assembled context: stored keys are R(p_orig) k; un-rotate, re-rotate at p_new
        kc = torch.cat([st.k[0, :, r:r + group_tok, :hd] for r in rows0[pick]], dim=1).double()  # [Hkv, T', hd]
        vc = torch.cat([st.v[0, :, :hd, r:r + group_tok] for r in rows0[pick]], dim=2).double().transpose(1, 2)
        p_orig = torch.cat([torch.arange(pos0[b], pos0[b] + group_tok, device=dev) for b in pick])
        k_pre = _rope64_t(kc, -p_orig, theta)
        k_asm = _rope64_t(k_pre, torch.arange(Tp, device=dev), theta)
        qn = qkv[t0:t0 + n, :qw].double().view(n, H, hd).transpose(0, 1)  # [H, n, hd]
        kn = qkv[t0:t0 + n, qw:qw + kw].double().view(n, Hkv, hd).transpose(0, 1)
        vn = qkv[t0:t0 + n, qw + kw:].double().view(n, Hkv, hd).transpose(0, 1)
        qr = _rope64_t(qn, pos, theta)
        kr = _rope64_t(kn, pos, theta)
        lo = torch.as_tensor(np.asarray(job.lo), device=dev)
        r_i = torch.arange(n, device=dev)[:, None]
        k_i = torch.arange(n, device=dev)[None, :]
        vis = (k_i <= r_i) & ((k_i < job.prefix) | (k_i >= lo[:, None]))
        K = torch.cat([k_asm, kr], dim=1)  # [Hkv, T'+n, hd]
        V = torch.cat([vc, vn], dim=1)
        mask = torch.cat([torch.ones(n, Tp, dtype=torch.bool, device=dev), vis], dim=1)
        for kv in range(Hkv):
            q = qr[kv * gs:(kv + 1) * gs]  # [gs, n, hd]
            s = (q @ K[kv].T) * scale
            s = torch.where(mask[None], s, -torch.inf)
            p_ = torch.softmax(s, dim=-1)
            want = p_ @ V[kv]  # [gs, n, hd]
            if mode == "chunk-last":  # the kept rows, compact in job order
                rows = out[koff[qi]:koff[qi + 1]].view(-1, H, hd)[:, kv * gs:(kv + 1) * gs].transpose(0, 1).double()
                want = want[:, torch.as_tensor(kept[qi], device=dev)]
                got = rows
            else:
                got = out[t0:t0 + n].view(n, H, hd)[:, kv * gs:(kv + 1) * gs].transpose(0, 1).double()
            worst = max(worst, float((got - want).abs().max()))
    return worst


def test_k3_at_c3_shape_vs_float64():
    """C3: Llama-3.1-8B heads (32 q / 8 kv, hd 128, theta 5e5), a 90k-token
    pool of 60 x 1,500-token groups, 18 groups per query (T' = 27,000, so 211
    key tiles per work stream and re-positioning deltas up to ~63k with rope
    rows up to 90k), 64 queries of 32 tokens + 4 labels x 4 tokens."""
    worst = _stage2_at_scale(32, 8, 128, 500000.0, 60, 1500, 18, 64, 32, (4, 4), check=[0, 17, 40, 63])
    assert worst < 2e-2, worst


def test_k3_last_layer_scored_rows_at_c3_shape_vs_float64():
    """The last layer's schedule (Stage2Plan.last: scored rows only, SELF works
    through the row map, compact merge output) at the C3 shape."""
    worst = _stage2_at_scale(32, 8, 128, 500000.0, 60, 1500, 18, 64, 32, (4, 4), check=[0, 17, 40, 63],
                             mode="chunk-last")
    assert worst < 2e-2, worst


@pytest.mark.parametrize("n_queries", [1, 3])
def test_k3_split_packed_at_c3_shape_vs_float64(n_queries):
    """Batch 1 (and 3) at the C3 shape through the split-KV schedule as
    Runner.infer runs it: cost-packed CTA ranges (DbsaAttnArgs.cta_works), the
    queries' own tokens as a split of their own, bf16 partials."""
    worst = _stage2_at_scale(32, 8, 128, 500000.0, 60, 1500, 18, n_queries, 32, (4, 4),
                             check=list(range(n_queries)), mode="query")
    assert worst < 2e-2, worst


def test_k3_at_c4_shape_vs_float64():
    """C4: Llama-2-7B MHA (32 heads, Hkv 32, hd 128, theta 1e4), 7 groups of
    4,096 tokens, 3 selected (T' = 12,288), 16 queries."""
    worst = _stage2_at_scale(32, 32, 128, 10000.0, 7, 4096, 3, 16, 32, (4, 4), check=[0, 9, 15])
    assert worst < 2e-2, worst


def _stage1_at_scale(H, Hkv, hd, theta, lengths, j=2, check_groups=None, seed=7):
    """One layer of K1 over whole groups (sink + prev-j + causal self,
    masks.py:80-99, 164-177) at a north-star shape against float64 attention
    over each group's allowed keys (torch on the GPU)."""
    dev = torch.device("cuda", 0)
    gs = H // Hkv
    T = sum(lengths)
    pos0 = np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)
    page0, p = [], 0
    for n in lengths:
        page0.append(p)
        p += -(-n // ops.PAGE)
    rows = p * ops.PAGE
    hdp = ops.hd_pad(hd)
    g = torch.Generator(device=dev).manual_seed(seed)
    k_pre = torch.randn(T, Hkv, hd, generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn(T, Hkv, hd, generator=g, device=dev).to(torch.bfloat16)
    q = torch.randn(T, H, hd, generator=g, device=dev).to(torch.bfloat16)
    kp = torch.zeros(1, Hkv, rows, hdp, dtype=torch.bfloat16, device=dev)
    vp = torch.zeros(1, Hkv, hdp, rows, dtype=torch.bfloat16, device=dev)
    rope = ops.rope_table(T + 64, hd, theta, dev)
    pages = []
    for b, n in enumerate(lengths):
        for i in range(0, n, ops.PAGE):
            pages.append((int(pos0[b]) + i, min(ops.PAGE, n - i), page0[b] * ops.PAGE + i, 0))
    pages = np.array(pages, dtype=np.int32).view(ops.PAGE_DTYPE).reshape(-1)
    pos = torch.arange(T, dtype=torch.int32, device=dev)
    ops.kv_write(k_pre.reshape(T, -1), v.reshape(T, -1), Hkv * hd, pos, rope, ops.to_device(pages, dev), len(pages),
                 kp, vp, rows, 1, 0, Hkv, hd)
    num_m = 2 if max(lengths) * gs > 128 else 1
    slab = (128 * num_m) // gs
    works, segs = [], []
    ctx_of = []
    for b, n in enumerate(lengths):
        ctx = sorted({0} | set(range(max(0, b - j), b)) - {b}) if b > 0 else []
        ctx_of.append(ctx)
        for kv in range(Hkv):
            for t0 in range(0, n, slab):
                nt = min(slab, n - t0)
                sb = len(segs)
                for c in ctx:
                    segs.append((0, 0, page0[c] * ops.PAGE, lengths[c], ops.nat.SEG_FULL, 0, 0, 0))
                segs.append((0, 0, page0[b] * ops.PAGE, t0 + nt, ops.nat.SEG_SELF, 0, 0, 0))
                works.append((int(pos0[b]) + t0, nt, int(pos0[b]), kv, sb, len(segs), 0, 0, 0))
    wa = np.zeros(len(works), dtype=ops.WORK_DTYPE)
    for i, name in enumerate(ops.WORK_DTYPE.names):
        wa[name] = [w[i] for w in works]
    sa = np.array(segs, dtype=np.int32).view(ops.SEG_DTYPE).reshape(-1)
    out = torch.zeros(T, H, hd, dtype=torch.bfloat16, device=dev)
    ops.attention(q=q, q_tok_stride=H * hd, tok_pos=pos, tok_lo=None, rope=rope, pool=(kp, vp, rows, 1), aux=None,
                  n_heads=H, n_kv_heads=Hkv, head_dim=hd, works_dev=ops.to_device(wa, dev), n_works=len(wa),
                  segs_dev=ops.to_device(sa, dev), num_m=num_m, out=out, out_tok_stride=H * hd)
    torch.cuda.synchronize()
    posd = torch.arange(T, device=dev)
    kr = _rope64_t(k_pre.double().transpose(0, 1), posd, theta)  # [Hkv, T, hd]
    qr = _rope64_t(q.double().transpose(0, 1), posd, theta)      # [H, T, hd]
    vv = v.double().transpose(0, 1)
    scale = 1.0 / math.sqrt(hd)
    worst = 0.0
    for b in (check_groups if check_groups is not None else range(len(lengths))):
        n, s0 = lengths[b], int(pos0[b])
        keys = torch.cat([torch.arange(pos0[c], pos0[c] + lengths[c], device=dev) for c in ctx_of[b]]
                         + [torch.arange(s0, s0 + n, device=dev)])
        n_ctx = keys.numel() - n
        mask = torch.ones(n, keys.numel(), dtype=torch.bool, device=dev)
        mask[:, n_ctx:] = torch.tril(torch.ones(n, n, dtype=torch.bool, device=dev))
        for kv in range(Hkv):
            qq = qr[kv * gs:(kv + 1) * gs, s0:s0 + n]
            s = (qq @ kr[kv, keys].T) * scale
            s = torch.where(mask[None], s, -torch.inf)
            want = torch.softmax(s, dim=-1) @ vv[kv, keys]
            got = out[s0:s0 + n, kv * gs:(kv + 1) * gs].transpose(0, 1).double()
            worst = max(worst, float((got - want).abs().max()))
    return worst


def test_k1_at_c2_shape_vs_float64():
    """C2: Llama-3.1-8B heads (32 / 8, hd 128, theta 5e5), 1,500-token groups,
    sink + prev-2 + self (groups 3.. see 4,500 context keys + causal self)."""
    worst = _stage1_at_scale(32, 8, 128, 500000.0, [1500] * 6, j=2, check_groups=[0, 1, 3, 5])
    assert worst < 2e-2, worst


def test_k1_at_c4_shape_vs_float64():
    """C4: MHA (gs 1) with 4,096-token groups, theta 1e4 (8 heads keep the
    float64 check quick; the per-head work is the C4 shape)."""
    worst = _stage1_at_scale(8, 8, 128, 10000.0, [4096] * 3, j=2)
    assert worst < 2e-2, worst


# ---------------------------------------------------------------- K5 fused label scoring
@pytest.mark.parametrize("rows,d,vocab", [(1, 64, 259), (5, 64, 259), (130, 512, 1000), (300, 200, 777),
                                          (13, 4096, 128256), (128, 4096, 128256), (832, 4096, 128256)])
def test_label_score_vs_float64(rows, d, vocab):
    """K5 (dbsa_label_score): log_softmax(x @ lm_head)[row, target] for scored
    (row, target) pairs without materialising logits, against float64 over
    the same bf16 operands (model.py:393-397, 414-417, 441-443).  Shapes: the
    C1 tokenizer vocab, a vocab that is not a multiple of the 256-column tile,
    a d that is not a multiple of the 64-wide K slice, rows past one and two M
    tiles, the batch-1 narrow form at the Llama-3 vocab (13 and 128 rows: N =
    128 vocab tiles, x loaded for its real rows), and the C3 batch (832
    distinct scored rows)."""
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(rows + d)
    x = (torch.randn(rows, d, generator=g, device=dev) * 2).to(torch.bfloat16)
    w = (torch.rand(vocab, d, generator=g, device=dev) * 2 - 1).mul(3.0 / d ** 0.5).to(torch.bfloat16)
    n_pairs = max(1, rows * 5 // 4)
    pair_row = torch.randint(0, rows, (n_pairs,), generator=g, device=dev)
    pair_tgt = torch.randint(0, vocab, (n_pairs,), generator=g, device=dev).to(torch.int32)
    pair_tgt[0] = vocab - 1  # the last column of a partial vocab tile
    lp = ops.label_score(x, w, pair_row, pair_tgt)
    torch.cuda.synchronize()
    ref = torch.log_softmax(x.double() @ w.double().T, dim=-1)[pair_row, pair_tgt.long()]
    err = float((lp.double() - ref).abs().max())
    assert err < 2e-3, err
