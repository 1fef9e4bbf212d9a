"""Device-op wrappers over the C ABI (torch tensors in, launches on the current
stream out).  Torch is used only for device memory and streams here; every
computation is one of the hand-written sm_100a kernels in csrc/.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from . import _native as nat
from .errors import ConfigError, ShapeError

PAGE = nat.PAGE_TOKENS

# Number of libdbsa kernel launches issued through this module (bench.py's
# `gpu_launches`).  Plain int: increments are GIL-atomic enough for a count.
LAUNCHES = 0


def _launched(n: int = 1) -> None:
    global LAUNCHES
    LAUNCHES += n


def _p(x) -> int:
    """Device pointer of a tensor, or an int address passed through."""
    return int(x) if isinstance(x, int) else int(x.data_ptr())

WORK_DTYPE = np.dtype(
    [("q_tok0", "<i4"), ("n_tok", "<i4"), ("self_tok0", "<i4"), ("kv_head", "<i4"),
     ("seg_begin", "<i4"), ("seg_end", "<i4"), ("prefix", "<i4"), ("out_mode", "<i4"),
     ("part_row0", "<i8")], align=True)
SEG_DTYPE = np.dtype(
    [("src", "<i4"), ("layer", "<i4"), ("row0", "<i4"), ("n_tok", "<i4"),
     ("kind", "<i4"), ("shift", "<i4"), ("pad0", "<i4"), ("pad1", "<i4")], align=True)
ROWMAP_DTYPE = np.dtype([("tok", "<i4"), ("rope_row", "<i4"), ("part_tok", "<i4"), ("pad", "<i4")], align=True)
PAGE_DTYPE = np.dtype([("tok0", "<i4"), ("n_tok", "<i4"), ("row0", "<i4"), ("pad", "<i4")], align=True)
MERGE_DTYPE = np.dtype(
    [("part_row0", "<i8"), ("rows", "<i4"), ("n_splits", "<i4"), ("q_tok0", "<i4"), ("kv_head", "<i4")],
    align=True)

assert WORK_DTYPE.itemsize == ctypes.sizeof(nat.AttnWork)
assert SEG_DTYPE.itemsize == ctypes.sizeof(nat.AttnSeg)
assert ROWMAP_DTYPE.itemsize == ctypes.sizeof(nat.RowMap)
assert PAGE_DTYPE.itemsize == ctypes.sizeof(nat.Page)
assert MERGE_DTYPE.itemsize == ctypes.sizeof(nat.MergeGroup)

ORDERING_CODES = {"in-order": 0, "low-to-high": 1, "reverse": 2}


def hd_pad(head_dim: int) -> int:
    """Head dim padded to a tcgen05-friendly width (zero columns)."""
    for p in (16, 32, 64, 128):
        if head_dim <= p:
            return p
    raise ConfigError(f"head_dim {head_dim} > 128 is not supported by the sm_100a kernels")


def inv_freq(head_dim: int, theta: float) -> np.ndarray:
    """theta ** (-arange(0, hd, 2) / hd) in float64 (model.rope_angles, model.py:207)."""
    return theta ** (-np.arange(0, head_dim, 2, dtype=np.float64) / head_dim)


def to_device(arr: np.ndarray, device):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8))
    if t.numel() == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return t.pin_memory().to(device, non_blocking=True)


def h2d(arr: np.ndarray, device):
    """Typed host array -> device tensor through pinned memory: the copy is
    stream-ordered and asynchronous (a pageable source would block the host
    until the stream's earlier work finished)."""
    import torch

    return torch.from_numpy(np.ascontiguousarray(arr)).pin_memory().to(device, non_blocking=True)


def rope_table(rows: int, head_dim: int, theta: float, device, pos0: int = 0):
    """float32 [rows, hd/2, 2] table of (cos, sin)(pos * inv_freq) built on device in float64."""
    import torch

    half = head_dim // 2
    freq = torch.from_numpy(inv_freq(head_dim, theta)).to(device)
    table = torch.empty((rows, half, 2), dtype=torch.float32, device=device)
    nat.check(nat.load_library().dbsa_rope_table(table.data_ptr(), rows, freq.data_ptr(), half, pos0,
                                                 nat.stream_handle()))
    _launched()
    table._keepalive = freq  # freq must outlive the async launch
    if os.environ.get("DBSA_ROPE_F16", "1") != "0":
        # fp16 copy for the attention kernels' query rotation (DbsaAttnArgs.rope_f16)
        table.f16 = torch.empty((rows, half, 2), dtype=torch.float16, device=device)
        nat.check(nat.load_library().dbsa_rope_table_f16(table.f16.data_ptr(), rows, freq.data_ptr(), half, pos0,
                                                         nat.stream_handle()))
        _launched()
    return table


def kv_write(k_src, v_src, src_tok_stride, tok_pos, rope, pages_dev, n_pages, k_dst, v_dst, dst_rows,
             dst_layers, layer, n_kv_heads, head_dim):
    a = nat.KvWriteArgs(
        k_src=k_src.data_ptr(), v_src=v_src.data_ptr(), src_tok_stride=src_tok_stride,
        tok_pos=tok_pos.data_ptr(), rope_table=rope.data_ptr(), rope_rows=rope.shape[0],
        pages=pages_dev.data_ptr(), n_pages=n_pages, k_dst=k_dst.data_ptr(), v_dst=v_dst.data_ptr(),
        dst_rows=dst_rows, dst_layers=dst_layers, layer=layer, n_kv_heads=n_kv_heads,
        head_dim=head_dim, hd_pad=hd_pad(head_dim))
    nat.check(nat.load_library().dbsa_kv_write(ctypes.byref(a), nat.stream_handle()))
    _launched()


def kv_read(k_planes, v_planes, rows, layers, layer, tok_pos, rope, pages_dev, n_pages, n_kv_heads, head_dim,
            k_dst, v_dst):
    """K2r: fp32 pre-rotation K and V (token-major) of a set of pages."""
    a = nat.KvReadArgs(k_src=k_planes.data_ptr(), v_src=v_planes.data_ptr(), src_rows=rows, src_layers=layers,
                       layer=layer, tok_pos=tok_pos.data_ptr(), rope_table=rope.data_ptr(), rope_rows=rope.shape[0],
                       pages=pages_dev.data_ptr(), n_pages=n_pages, n_kv_heads=n_kv_heads, head_dim=head_dim,
                       hd_pad=hd_pad(head_dim), k_dst=k_dst.data_ptr(), v_dst=v_dst.data_ptr())
    nat.check(nat.load_library().dbsa_kv_read(ctypes.byref(a), nat.stream_handle()))
    _launched()


PART_CHUNKED = os.environ.get("DBSA_PART_CHUNKED", "1") != "0"


def chunk_rows_of(part_o, head_dim: int) -> int:
    """DbsaAttnArgs / DbsaMergeArgs.part_chunk_rows of a partial buffer: bf16
    [rows, head_dim] buffers use the 16-column chunk layout (rows = the
    buffer's first dimension, so the K3 launch that writes it and the K3m that
    reads it agree); anything else is row-major."""
    if not PART_CHUNKED or part_o is None or part_o.dim() != 2 or part_o.element_size() != 2 or head_dim % 16:
        return 0
    return int(part_o.shape[0])


def attention(*, q, q_tok_stride, tok_pos, tok_lo, rope, pool, aux, n_heads, n_kv_heads, head_dim,
              works_dev, n_works, segs_dev, num_m, out, out_tok_stride, part_o=None, part_lse=None,
              row_map=None, pair_count=None, cta_works=None, n_ctas=0, after_kv_write=False,
              part_chunk_rows=None, one_seg_partials=False):
    """Launch K1/K3.  `pool` / `aux` are (k_planes, v_planes, rows, layers); `row_map`
    (ROWMAP_DTYPE, device) backs DBSA_OUT_MAPPED works; `pair_count` (int64 [1],
    device) makes the kernel add the (row, key) pairs it unmasked, all heads;
    `cta_works` (int32 [n_ctas + 1], device) assigns CTA b the works
    [cta_works[b], cta_works[b+1]) (two-tile kernel only); after_kv_write: the
    launch directly follows the layer's K2w page write, so Q staging may
    overlap it (DbsaAttnArgs.pdl_early_q); part_chunk_rows: the partials'
    layout (None = chunk_rows_of(part_o)); one_seg_partials: every work has
    one segment and writes a partial (the chunk-major schedule), which allows
    the specialised kernel instance (DbsaAttnArgs.one_seg_partials)."""
    kp, vp, prow, pl = pool
    ka, va, arow, al = aux if aux is not None else (None, None, 0, 0)
    a = nat.AttnArgs(
        q=q.data_ptr(), q_tok_stride=q_tok_stride, tok_pos=tok_pos.data_ptr(),
        tok_lo=nat.ptr(tok_lo), rope_table=rope.data_ptr(), rope_rows=rope.shape[0],
        k_pool=kp.data_ptr(), v_pool=vp.data_ptr(), pool_rows=prow,
        pool_layers=pl, k_aux=nat.ptr(ka), v_aux=nat.ptr(va), aux_rows=arow, aux_layers=al,
        n_heads=n_heads, n_kv_heads=n_kv_heads, head_dim=head_dim, hd_pad=hd_pad(head_dim),
        scale=float(1.0 / math.sqrt(head_dim)), num_m=num_m, works=_p(works_dev),
        n_works=n_works, segs=_p(segs_dev), out=out.data_ptr(), out_tok_stride=out_tok_stride,
        part_o=nat.ptr(part_o), part_lse=nat.ptr(part_lse), row_map=nat.ptr(row_map),
        part_bf16=int(part_o is not None and part_o.element_size() == 2), pair_count=nat.ptr(pair_count),
        cta_works=nat.ptr(cta_works), n_ctas=int(n_ctas), pdl_early_q=int(bool(after_kv_write)),
        rope_f16=nat.ptr(getattr(rope, "f16", None)),
        part_chunk_rows=chunk_rows_of(part_o, head_dim) if part_chunk_rows is None else part_chunk_rows,
        one_seg_partials=int(bool(one_seg_partials)))
    nat.check(nat.load_library().dbsa_attention(ctypes.byref(a), nat.stream_handle()))
    _launched()


def lse_merge(part_o, part_lse, groups_dev, n_groups, max_rows, n_heads, n_kv_heads, head_dim, out,
              out_tok_stride, split_stride=0, out_lse=None, tok_layout=False, part_chunk_rows=None):
    """K3m.  out_lse (fp32 [tokens, n_heads], device): write the merged partial
    (bf16 O into `out`, its LSE into out_lse) instead of the final output;
    tok_layout: the partials are token-major [split][tokens][n_heads][hd] (a
    gathered set of out_lse-mode results, split_stride = tokens * n_heads)."""
    a = nat.MergeArgs(part_o=part_o.data_ptr(), part_lse=part_lse.data_ptr(), groups=groups_dev.data_ptr(),
                      n_groups=n_groups, max_rows=max_rows, n_heads=n_heads, n_kv_heads=n_kv_heads,
                      head_dim=head_dim, out=out.data_ptr(), out_tok_stride=out_tok_stride,
                      split_stride=split_stride, part_bf16=int(part_o.element_size() == 2),
                      part_tok_layout=int(bool(tok_layout)), out_lse=nat.ptr(out_lse),
                      part_chunk_rows=(0 if tok_layout else chunk_rows_of(part_o, head_dim))
                      if part_chunk_rows is None else part_chunk_rows)
    nat.check(nat.load_library().dbsa_lse_merge(ctypes.byref(a), nat.stream_handle()))
    _launched()


def topk_select(scores, budget: int, ordering: str):
    """scores: float64 [n_queries, n_units] (device) -> int32 [n_queries, budget] unit ids."""
    import torch

    if scores.dtype != torch.float64 or scores.dim() != 2:
        raise ShapeError("topk_select expects a 2-D float64 score matrix")
    scores = scores.contiguous()
    out = torch.empty((scores.shape[0], budget), dtype=torch.int32, device=scores.device)
    nat.check(nat.load_library().dbsa_topk_select(
        scores.data_ptr(), scores.shape[0], scores.shape[1], budget, ORDERING_CODES[ordering],
        out.data_ptr(), nat.stream_handle()))
    _launched()
    return out


def rmsnorm(x, weight, eps: float, out=None):
    import torch

    out = out if out is not None else torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    nat.check(nat.load_library().dbsa_rmsnorm(x.data_ptr(), weight.data_ptr(), out.data_ptr(), x.shape[0],
                                              x.shape[1], float(eps), nat.stream_handle()))
    _launched()
    return out


def add_rmsnorm(x, delta, weight, eps: float, out):
    """x += delta (fp32, in place); out = bf16 RMSNorm(x) * weight."""
    nat.check(nat.load_library().dbsa_add_rmsnorm(x.data_ptr(), delta.data_ptr(), weight.data_ptr(), out.data_ptr(),
                                                  x.shape[0], x.shape[1], float(eps), nat.stream_handle()))
    _launched()
    return out


def silu_mul(gate_up, ffn: int, out=None):
    import torch

    out = out if out is not None else torch.empty((gate_up.shape[0], ffn), dtype=torch.bfloat16,
                                                  device=gate_up.device)
    nat.check(nat.load_library().dbsa_silu_mul(gate_up.data_ptr(), out.data_ptr(), gate_up.shape[0], ffn,
                                               nat.stream_handle()))
    _launched()
    return out


def label_logprob(logits, targets):
    import torch

    out = torch.empty(logits.shape[0], dtype=torch.float32, device=logits.device)
    nat.check(nat.load_library().dbsa_label_logprob(logits.data_ptr(), logits.shape[0], logits.shape[1],
                                                     targets.data_ptr(), out.data_ptr(), nat.stream_handle()))
    _launched()
    return out


def label_score_workspace_shape(rows: int, vocab: int) -> tuple[int, int, int]:
    """fp32 [vocab / 128][rows rounded up to 128][(max, sum)] of K5."""
    return (-(-vocab // 128), -(-rows // 128) * 128, 2)


def label_score(x, lm_head_t, pair_row, pair_target, workspace=None, out=None):
    """K5 (dbsa_label_score): log p(target | row) of every scored pair, from the
    final-normed rows x (bf16 [rows, d]) and the K-major lm_head (bf16
    [vocab, d]), without materialising logits."""
    import torch

    rows, d = x.shape
    vocab = lm_head_t.shape[0]
    shape = label_score_workspace_shape(rows, vocab)
    if workspace is None or tuple(workspace.shape) != shape:
        workspace = torch.empty(shape, dtype=torch.float32, device=x.device)
    n = pair_row.numel()
    out = out if out is not None else torch.empty(n, dtype=torch.float32, device=x.device)
    a = nat.LabelScoreArgs(x=x.data_ptr(), rows=rows, d=d, w=lm_head_t.data_ptr(), vocab=vocab,
                           workspace=workspace.data_ptr(), pair_row=pair_row.data_ptr(),
                           pair_target=pair_target.data_ptr(), n_pairs=n, out=out.data_ptr())
    nat.check(nat.load_library().dbsa_label_score(ctypes.byref(a), nat.stream_handle()))
    _launched(2)
    return out


def label_reduce(lp, label_row0, n_queries: int, n_labels: int):
    """Per-label sums of token log-probs and the first-max label per query."""
    import torch

    scores = torch.empty((n_queries, n_labels), dtype=torch.float32, device=lp.device)
    best = torch.empty(n_queries, dtype=torch.int64, device=lp.device)
    nat.check(nat.load_library().dbsa_label_reduce(lp.data_ptr(), label_row0.data_ptr(), n_queries, n_labels,
                                                    scores.data_ptr(), best.data_ptr(), nat.stream_handle()))
    _launched()
    return scores, best


def bm25_scores(term_ids, tf, idf, norm, k1p1: float):
    """term_ids int32 [Q, T] (-1 pad), tf uint16 [V, U], idf f64 [V], norm f64 [U] -> f64 [Q, U]."""
    import torch

    n_q, max_terms = term_ids.shape
    n_units = tf.shape[1]
    out = torch.empty((n_q, n_units), dtype=torch.float64, device=tf.device)
    nat.check(nat.load_library().dbsa_bm25_scores(term_ids.data_ptr(), n_q, max_terms, tf.data_ptr(), idf.data_ptr(),
                                                   norm.data_ptr(), n_units, float(k1p1), out.data_ptr(),
                                                   nat.stream_handle()))
    _launched()
    return out
