"""CPU oracle for the DBSA hot path -- TEST INFRASTRUCTURE ONLY.

A numpy / pure-Python restatement of the reference algorithm (the package at
/root/reference/pkg/src/dbsa, read-only, Python 3.12 + numpy).  Each function
cites the reference file:line it follows.  It is used ONLY by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg,
as the checker or the timed CPU baseline -- never by the product path
(paper_2503_08640_b200/), which must fail loudly without its CUDA library.

Parity pinning: tests/golden/make_golden.py imported the reference itself in
the build container and recorded golden vectors (tests/golden/*.npz);
tests/test_oracle_golden.py checks this oracle against them (weights
checksum, partition, block mask, pair counts, K/V samples, BM25 scores,
selected unit ids, label scores, logits).

Numerics follow the reference exactly: float32 storage with float64
accumulation and a single float32 rounding at the same points
(kernels.py:1-7): matmul, rms_norm, silu_gate, rope, attention outputs, and
the float64 residual adds of model.py:353,359.
"""

from __future__ import annotations

import hashlib
import math
import re
from collections import Counter
from dataclasses import dataclass

import numpy as np

F32 = np.float32

# ----------------------------------------------------------------- tokenizer
BYTE_OFFSET = 3  # tokenizer.py:10-13
VOCAB = 256 + BYTE_OFFSET


def encode(text: str) -> list[int]:
    """Byte-level ids, byte + 3 (tokenizer.py:17-18)."""
    return [b + BYTE_OFFSET for b in text.encode("utf-8")]


def make_rng(seed: int) -> np.random.Generator:
    """Philox-backed generator (kernels.py:126-130)."""
    return np.random.Generator(np.random.Philox(int(seed)))


# ----------------------------------------------------------------- config / weights
@dataclass(frozen=True)
class Cfg:
    d_model: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab_size: int = VOCAB
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    max_seq_len: int = 32768

    @property
    def gs(self) -> int:
        return self.n_heads // self.n_kv_heads


def weight_shapes(c: Cfg) -> dict[str, tuple[int, ...]]:
    """(in, out) layout, x @ W (model.py:103-126)."""
    s = {"tok_embed": (c.vocab_size, c.d_model), "out_norm": (c.d_model,), "lm_head": (c.d_model, c.vocab_size)}
    q, kv = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
    for i in range(c.n_layers):
        p = f"layers.{i}."
        s |= {p + "attn_norm": (c.d_model,), p + "wq": (c.d_model, q), p + "wk": (c.d_model, kv),
              p + "wv": (c.d_model, kv), p + "wo": (q, c.d_model), p + "ffn_norm": (c.d_model,),
              p + "w_gate": (c.d_model, c.ffn_dim), p + "w_up": (c.d_model, c.ffn_dim),
              p + "w_down": (c.ffn_dim, c.d_model)}
    return s


def init_random(c: Cfg, seed: int) -> dict[str, np.ndarray]:
    """Scaled-uniform init in sorted-name order from one Philox stream (model.py:159-171)."""
    rng = make_rng(seed)
    w = {}
    for name, shape in sorted(weight_shapes(c).items()):
        if name.endswith("norm"):
            w[name] = np.ones(shape, F32)
        elif name == "tok_embed":
            w[name] = rng.uniform(-0.1, 0.1, size=shape).astype(F32)
        else:
            lim = 1.0 / np.sqrt(shape[0])
            w[name] = rng.uniform(-lim, lim, size=shape).astype(F32)
    return w


def weights_checksum(w: dict[str, np.ndarray]) -> str:
    """sha256 over sorted (name, f32 bytes) (model.py:151-156)."""
    h = hashlib.sha256()
    for name in sorted(w):
        h.update(name.encode())
        h.update(np.ascontiguousarray(w[name], F32).tobytes())
    return h.hexdigest()


# ----------------------------------------------------------------- numerics
def mm(a, b):
    """f64 product rounded to f32 (kernels.py:31-40)."""
    return (np.asarray(a, np.float64) @ np.asarray(b, np.float64)).astype(F32)


def rms_norm(x, g, eps):
    """kernels.py:103-112."""
    x = np.asarray(x, np.float64)
    return (x / np.sqrt((x * x).mean(-1, keepdims=True) + eps) * np.asarray(g, np.float64)).astype(F32)


def silu_gate(g, u):
    """kernels.py:115-123."""
    g = np.asarray(g, np.float64)
    return (g / (1.0 + np.exp(-g)) * np.asarray(u, np.float64)).astype(F32)


def rope(x, positions, theta):
    """Paired-halves rotation of (T, heads, hd) at per-token positions, f64
    angles, f32 output (model.py:205-239)."""
    x = np.asarray(x, np.float64)
    hd = x.shape[-1]
    freq = theta ** (-np.arange(0, hd, 2, dtype=np.float64) / hd)
    ang = np.asarray(positions, np.float64)[:, None] * freq[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    a, b = x[..., : hd // 2], x[..., hd // 2:]
    return np.concatenate([a * c - b * s, a * s + b * c], axis=-1).astype(F32)


def masked_attention(q_scaled, k, v, mask):
    """softmax over allowed entries (f64, max-subtracted, masked exactly 0) then
    P @ V, rounded once to f32 (kernels.py:43-57, 73-100)."""
    mask = np.asarray(mask, bool)
    if not mask.any(axis=1).all():
        raise ValueError("masked softmax: a row has no allowed entries")
    s = np.asarray(q_scaled, np.float64) @ np.asarray(k, np.float64).T
    mx = np.max(s, axis=1, keepdims=True, where=mask, initial=-np.inf)
    e = np.where(mask, np.exp(np.where(mask, s - mx, 0.0)), 0.0)
    e /= e.sum(axis=1, keepdims=True)
    return (e @ np.asarray(v, np.float64)).astype(F32)


def forward(c: Cfg, w, ids, positions, ctx_pos, ctx_layers, mask):
    """Decoder body (model.py:282-360): returns per-layer PRE-rotation (K, V) of
    the new tokens and their final hidden states.  ctx_layers[l] = (K rotated
    at ctx_pos, V), shapes (n_ctx, Hkv, hd)."""
    ids = np.asarray(ids, np.int64)
    pos = np.asarray(positions, np.int64)
    t = len(ids)
    n_ctx = len(ctx_pos)
    mask = np.asarray(mask, bool)
    assert mask.shape == (t, n_ctx + t)
    scale = 1.0 / np.sqrt(c.head_dim)
    gmask = np.vstack([mask] * c.gs)  # heads of one kv group stacked head-major (model.py:336)
    h = w["tok_embed"][ids]
    kv_out = []
    for layer in range(c.n_layers):
        p = f"layers.{layer}."
        x = rms_norm(h, w[p + "attn_norm"], c.norm_eps)
        q = mm(x, w[p + "wq"]).reshape(t, c.n_heads, c.head_dim)
        k = mm(x, w[p + "wk"]).reshape(t, c.n_kv_heads, c.head_dim)
        v = mm(x, w[p + "wv"]).reshape(t, c.n_kv_heads, c.head_dim)
        kv_out.append((k.copy(), v.copy()))
        qr, kr = rope(q, pos, c.rope_theta), rope(k, pos, c.rope_theta)
        ck, cv = ctx_layers[layer] if n_ctx else (None, None)
        ka = np.concatenate([ck, kr]) if n_ctx else kr
        va = np.concatenate([cv, v]) if n_ctx else v
        att = np.empty((t, c.n_heads, c.head_dim), F32)
        for g in range(c.n_kv_heads):
            hs = slice(g * c.gs, (g + 1) * c.gs)
            qg = qr[:, hs, :].transpose(1, 0, 2).reshape(c.gs * t, c.head_dim)
            o = masked_attention((qg * scale).astype(F32), ka[:, g], va[:, g], gmask)
            att[:, hs, :] = o.reshape(c.gs, t, c.head_dim).transpose(1, 0, 2)
        h = (h.astype(np.float64) + mm(att.reshape(t, -1), w[p + "wo"]).astype(np.float64)).astype(F32)
        x = rms_norm(h, w[p + "ffn_norm"], c.norm_eps)
        f = mm(silu_gate(mm(x, w[p + "w_gate"]), mm(x, w[p + "w_up"])), w[p + "w_down"])
        h = (h.astype(np.float64) + f.astype(np.float64)).astype(F32)
    return kv_out, h


def logits(c: Cfg, w, hidden):
    """model.py:395-397."""
    return mm(rms_norm(hidden, w["out_norm"], c.norm_eps), w["lm_head"])


def log_softmax_rows(z):
    """f64 log-softmax (model.py:414-417)."""
    z = np.asarray(z, np.float64)
    z = z - z.max(axis=1, keepdims=True)
    return z - np.log(np.exp(z).sum(axis=1, keepdims=True))


def query_mask(n_ctx, t):
    """Full context + causal self (model.py:381-384)."""
    m = np.ones((t, n_ctx + t), bool)
    m[:, n_ctx:] = np.tril(np.ones((t, t), bool))
    return m


def forward_query(c: Cfg, w, asm_layers, n_ctx, query_ids):
    """Logits of every query position against an assembled cache (model.py:400-411)."""
    pos = np.arange(n_ctx, n_ctx + len(query_ids))
    _, h = forward(c, w, query_ids, pos, np.arange(n_ctx), asm_layers, query_mask(n_ctx, len(query_ids)))
    return logits(c, w, h)


def score_label(c: Cfg, w, asm_layers, n_ctx, query_ids, label_ids):
    """Teacher-forced sum of label log-probs (model.py:420-443)."""
    seq = list(query_ids) + list(label_ids)
    pos = np.arange(n_ctx, n_ctx + len(seq))
    _, h = forward(c, w, seq, pos, np.arange(n_ctx), asm_layers, query_mask(n_ctx, len(seq)))
    lp = log_softmax_rows(logits(c, w, h)[len(query_ids) - 1: len(seq) - 1])
    return float(lp[np.arange(len(label_ids)), label_ids].sum())


# ----------------------------------------------------------------- masks
def block_mask(n_blocks: int, kind: str, j: int = 2) -> np.ndarray:
    """Lower-triangular allowed[i, j] for full / sink-prev-self(j) / sink-self /
    self (masks.py:80-99)."""
    b = n_blocks
    if kind == "full":
        return np.tril(np.ones((b, b), bool))
    a = np.eye(b, dtype=bool)
    if kind in ("sink-self", "sink-prev-self"):
        a[:, 0] = True
    if kind == "sink-prev-self":
        for i in range(1, b):
            a[i, max(0, i - j): i] = True
    return np.tril(a)


def context_ids(allowed: np.ndarray, i: int) -> tuple[int, ...]:
    """Allowed context blocks of i, ascending, excluding i (masks.py:74-77)."""
    return tuple(int(x) for x in np.flatnonzero(allowed[i]) if x < i)


def allowed_token_pairs(allowed: np.ndarray, counts) -> int:
    """Causal self pairs + full cross pairs (masks.py:111-123)."""
    counts = [int(x) for x in counts]
    tot = sum(t * (t + 1) // 2 for t in counts)
    for i in range(len(counts)):
        for k in range(i):
            if allowed[i, k]:
                tot += counts[i] * counts[k]
    return tot


def full_token_mask(allowed, counts):
    """Dense (T, T) expansion (masks.py:149-161)."""
    off = np.concatenate([[0], np.cumsum(counts)]).astype(int)
    m = np.zeros((off[-1], off[-1]), bool)
    for i in range(len(counts)):
        m[off[i]:off[i + 1], off[i]:off[i + 1]] = np.tril(np.ones((counts[i], counts[i]), bool))
        for k in range(i):
            if allowed[i, k]:
                m[off[i]:off[i + 1], off[k]:off[k + 1]] = True
    return m


# ----------------------------------------------------------------- pool rendering / grouping
DEMO_FMT = "Q: {query}\nA: {answer}\n\n"  # pipeline.py:58-71
QUERY_FMT = "Q: {query}\nA:"
LABEL_FMT = " {label}"


def render_block(pool, members):
    """Block text, ids, per-demo spans (pipeline.py:149-163); pool = [(query, answer)]."""
    parts, spans, off = [], [], 0
    for e in members:
        part = DEMO_FMT.format(query=pool[e][0], answer=pool[e][1])
        n = len(encode(part))
        spans.append((off, off + n))
        off += n
        parts.append(part)
    text = "".join(parts)
    return text, encode(text), tuple(spans)


def random_partition(n: int, block_size: int, seed: int):
    """Random grouping: Philox permutation chunked (retrieval.py:322-334)."""
    order = [int(i) for i in make_rng(seed).permutation(n)]
    return [tuple(order[i:i + block_size]) for i in range(0, n, block_size)]


# ----------------------------------------------------------------- stage 1
def encode_blocks(c: Cfg, w, blocks_ids, kind="sink-prev-self", j=2):
    """Sequential stage-1 encode (pipeline.py:166-233): each block attends to
    its allowed context blocks, rotated at their ORIGINAL positions, and itself
    causally.  Returns (kv[layer][block] = (K_pre, V), attended pairs)."""
    counts = [len(x) for x in blocks_ids]
    off = np.concatenate([[0], np.cumsum(counts)]).astype(int)
    allowed = block_mask(len(counts), kind, j)
    kv = [[None] * len(counts) for _ in range(c.n_layers)]
    rot_cache = {}
    attended = 0
    for b, ids in enumerate(blocks_ids):
        ctx = context_ids(allowed, b)
        for cb in ctx:
            if cb not in rot_cache:
                p = np.arange(off[cb], off[cb + 1])
                rot_cache[cb] = [(rope(kv[l][cb][0], p, c.rope_theta), kv[l][cb][1]) for l in range(c.n_layers)]
        ctx_pos = np.concatenate([np.arange(off[cb], off[cb + 1]) for cb in ctx]) if ctx else np.zeros(0, int)
        ctx_layers = [(np.concatenate([rot_cache[cb][l][0] for cb in ctx]),
                       np.concatenate([rot_cache[cb][l][1] for cb in ctx])) if ctx else None
                      for l in range(c.n_layers)]
        t = len(ids)
        m = np.zeros((t, len(ctx_pos) + t), bool)
        m[:, :len(ctx_pos)] = True
        m[:, len(ctx_pos):] = np.tril(np.ones((t, t), bool))
        pre, _ = forward(c, w, ids, np.arange(off[b], off[b] + t), ctx_pos, ctx_layers, m)
        for l in range(c.n_layers):
            kv[l][b] = pre[l]
        attended += len(ctx_pos) * t + t * (t + 1) // 2
    return kv, attended


# ----------------------------------------------------------------- retrieval
_TERM = re.compile(r"[^\W_]+", re.UNICODE)


def bm25_terms(text: str) -> list[str]:
    """retrieval.py:41-43."""
    return _TERM.findall(text.lower())


class Bm25:
    """BM25 statistics and f64 scoring, k1=1.2, b=0.75 (retrieval.py:88-141)."""

    def __init__(self, texts, k1=1.2, b=0.75):
        self.k1, self.b = k1, b
        self.tf = [Counter(bm25_terms(t)) for t in texts]
        self.dl = [sum(c.values()) for c in self.tf]
        self.n = len(texts)
        self.avgdl = sum(self.dl) / self.n
        self.df = Counter(term for c in self.tf for term in c)

    def idf(self, term):
        d = self.df.get(term, 0)
        return math.log(1.0 + (self.n - d + 0.5) / (d + 0.5))

    def score(self, terms, doc):
        tf, dl = self.tf[doc], self.dl[doc]
        norm = self.k1 * (1.0 - self.b + self.b * dl / self.avgdl)
        acc = 0.0
        for term in terms:
            f = tf.get(term, 0)
            if f:
                acc += self.idf(term) * f * (self.k1 + 1.0) / (f + norm)
        return acc


def unit_texts(pool, partition, spans, granularity):
    """Unit texts and cache refs (block, start, end) per granularity (pipeline.py:236-262)."""
    raw = [f"{q} {a}" for q, a in pool]
    if granularity == "block":
        return ([" ".join(raw[e] for e in m) for m in partition],
                [(b, 0, spans[b][-1][1]) for b in range(len(partition))])
    texts = [" ".join(raw[e] for e in partition[0])]
    refs = [(0, 0, spans[0][-1][1])]
    for b in range(1, len(partition)):
        for slot, e in enumerate(partition[b]):
            texts.append(raw[e])
            refs.append((b, *spans[b][slot]))
    return texts, refs


def select(scores, ratio):
    """[0] + top-(budget-1) of 1..n-1 by (-score, id) (retrieval.py:352-374)."""
    n = len(scores)
    budget = math.ceil(ratio * n)
    return [0] + sorted(range(1, n), key=lambda u: (-scores[u], u))[: budget - 1]


def order(units, scores, strategy):
    """Anchor pinned; in-order / low-to-high / reverse (retrieval.py:377-388)."""
    rest = list(units[1:])
    if strategy == "in-order":
        rest.sort()
    elif strategy == "low-to-high":
        rest.sort(key=lambda u: (scores[u], u))
    else:
        rest.sort(key=lambda u: -u)
    return [units[0]] + rest


# ----------------------------------------------------------------- stage 2
def assemble(c: Cfg, kv, refs_sel):
    """Concatenate selected (block, start, end) spans, rotate K at new positions
    0..T'-1 (kvstore.py:188-221).  Returns (layers, T')."""
    total = sum(e - s for _, s, e in refs_sel)
    pos = np.arange(total)
    layers = []
    for l in range(c.n_layers):
        k = np.concatenate([kv[l][b][0][s:e] for b, s, e in refs_sel])
        v = np.concatenate([kv[l][b][1][s:e] for b, s, e in refs_sel])
        layers.append((rope(k, pos, c.rope_theta), v.copy()))
    return layers, total


def infer(c: Cfg, w, kv, index: Bm25, refs, labels, query_text, ratio=0.3, ordering="in-order"):
    """Runner.infer, DBSA branch (pipeline.py:389-421, 369-384): returns
    (label, per-label scores, ordered unit ids, T')."""
    terms = bm25_terms(query_text)
    scores = [index.score(terms, u) for u in range(index.n)]
    units = order(select(scores, ratio), scores, ordering)
    asm, n_ctx = assemble(c, kv, [refs[u] for u in units])
    q_ids = encode(QUERY_FMT.format(query=query_text))
    labs = sorted(labels)
    best, best_s, all_s = None, -np.inf, []
    for lab in labs:
        s = score_label(c, w, asm, n_ctx, q_ids, encode(LABEL_FMT.format(label=lab)))
        all_s.append(s)
        if s > best_s:
            best, best_s = lab, s
    return best, all_s, units, n_ctx


# ----------------------------------------------------------------- synthetic task
LABEL_WORDS = ("alpha", "bravo", "carol", "delta", "echo", "fox", "golf", "hotel",
               "india", "jazz", "kilo", "lima", "mike", "nova", "oscar", "papa")  # synthetic.py:13-16
FILLER = ("please", "kindly", "record", "note", "check", "confirm", "review",
          "item", "entry", "ticket", "case", "fact")


def recall_task(n_demos, n_tests, n_labels=4, seed=0):
    """Key -> label associative recall (synthetic.py:33-67).  Returns
    (pool [(q, a)], tests [(q, a)], labels)."""
    rng = make_rng(seed)
    labels = LABEL_WORDS[:n_labels]
    n_keys = max(4, n_demos // 3)
    key_label = {f"key{k:04d}": labels[int(rng.integers(n_labels))] for k in range(n_keys)}
    keys = list(key_label)

    def query(key):
        a = FILLER[int(rng.integers(len(FILLER)))]
        b = FILLER[int(rng.integers(len(FILLER)))]
        return f"{a} {b} lookup {key}"

    pool, used = [], []
    for i in range(n_demos):
        key = keys[int(rng.integers(n_keys))] if i >= n_keys else keys[i % n_keys]
        used.append(key)
        pool.append((query(key), key_label[key]))
    tests = []
    for _ in range(n_tests):
        key = used[int(rng.integers(len(used)))]
        tests.append((query(key), key_label[key]))
    return pool, tests, labels


def encode_pool(c: Cfg, w, pool, block_size, seed=0, kind="sink-prev-self", j=2, granularity="block"):
    """Stage 1 end to end (pipeline.py:286-319, random grouping): returns
    (partition, kv, attended, Bm25 index, unit refs, block token counts)."""
    partition = random_partition(len(pool), block_size, seed)
    rendered = [render_block(pool, m) for m in partition]
    kv, attended = encode_blocks(c, w, [ids for _, ids, _ in rendered], kind, j)
    texts, refs = unit_texts(pool, partition, [sp for _, _, sp in rendered], granularity)
    return partition, kv, attended, Bm25(texts), refs, [len(ids) for _, ids, _ in rendered]
