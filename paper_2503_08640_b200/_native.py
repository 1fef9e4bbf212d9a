"""ctypes binding of libdbsa_sm100a.so (include/dbsa_b200.h).

The library is the only compute backend of this package: there is no CPU or
eager fallback.  If the shared object is missing or no CUDA device is present
every compute entry point raises.  Non-zero return codes are mapped onto the
reference exception hierarchy (errors.py:4-29 of the reference package).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "libdbsa_sm100a.so"
if os.environ.get("DBSA_LIB"):  # kernel A/B experiments (tools/build_variant.py): an alternative build
    LIB_PATH = Path(os.environ["DBSA_LIB"])

EXPORTED_SYMBOLS = (
    "dbsa_attention",
    "dbsa_lse_merge",
    "dbsa_kv_write",
    "dbsa_kv_read",
    "dbsa_rope_table",
    "dbsa_topk_select",
    "dbsa_rmsnorm",
    "dbsa_add_rmsnorm",
    "dbsa_silu_mul",
    "dbsa_label_logprob",
    "dbsa_label_reduce",
    "dbsa_label_score",
    "dbsa_bm25_scores",
    "dbsa_abi_version",
    "dbsa_rope_table_f16",
    "dbsa_last_error",
)

ABI_VERSION = 12
OUT_BF16, OUT_PARTIAL, OUT_MAPPED = 0, 1, 2
PAGE_TOKENS = 64
SEG_FULL = 0
SEG_SELF = 1

_i32, _i64, _f32, _vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p


class AttnWork(ctypes.Structure):
    _fields_ = [
        ("q_tok0", _i32), ("n_tok", _i32), ("self_tok0", _i32), ("kv_head", _i32),
        ("seg_begin", _i32), ("seg_end", _i32), ("prefix", _i32), ("out_mode", _i32),
        ("part_row0", _i64),
    ]


class AttnSeg(ctypes.Structure):
    _fields_ = [
        ("src", _i32), ("layer", _i32), ("row0", _i32), ("n_tok", _i32),
        ("kind", _i32), ("shift", _i32), ("pad0", _i32), ("pad1", _i32),
    ]


class AttnArgs(ctypes.Structure):
    _fields_ = [
        ("q", _vp), ("q_tok_stride", _i64), ("tok_pos", _vp), ("tok_lo", _vp),
        ("rope_table", _vp), ("rope_rows", _i64),
        ("k_pool", _vp), ("v_pool", _vp), ("pool_rows", _i64), ("pool_layers", _i32),
        ("k_aux", _vp), ("v_aux", _vp), ("aux_rows", _i64), ("aux_layers", _i32),
        ("n_heads", _i32), ("n_kv_heads", _i32), ("head_dim", _i32), ("hd_pad", _i32),
        ("scale", _f32), ("num_m", _i32),
        ("works", _vp), ("n_works", _i32), ("segs", _vp),
        ("out", _vp), ("out_tok_stride", _i64), ("part_o", _vp), ("part_lse", _vp),
        ("row_map", _vp), ("part_bf16", _i32), ("pair_count", _vp), ("cta_works", _vp), ("n_ctas", _i32), ("pdl_early_q", _i32),
        ("rope_f16", _vp), ("part_chunk_rows", _i64), ("one_seg_partials", _i32),
    ]


class RowMap(ctypes.Structure):
    _fields_ = [("tok", _i32), ("rope_row", _i32), ("part_tok", _i32), ("pad", _i32)]


class MergeGroup(ctypes.Structure):
    _fields_ = [("part_row0", _i64), ("rows", _i32), ("n_splits", _i32), ("q_tok0", _i32), ("kv_head", _i32)]


class MergeArgs(ctypes.Structure):
    _fields_ = [
        ("part_o", _vp), ("part_lse", _vp), ("groups", _vp), ("n_groups", _i32), ("max_rows", _i32),
        ("n_heads", _i32), ("n_kv_heads", _i32), ("head_dim", _i32), ("out", _vp), ("out_tok_stride", _i64),
        ("split_stride", _i64), ("part_bf16", _i32), ("part_tok_layout", _i32), ("out_lse", _vp),
        ("part_chunk_rows", _i64),
    ]


class LabelScoreArgs(ctypes.Structure):
    _fields_ = [
        ("x", _vp), ("rows", _i64), ("d", _i64), ("w", _vp), ("vocab", _i64), ("workspace", _vp),
        ("pair_row", _vp), ("pair_target", _vp), ("n_pairs", _i64), ("out", _vp),
    ]


class Page(ctypes.Structure):
    _fields_ = [("tok0", _i32), ("n_tok", _i32), ("row0", _i32), ("pad", _i32)]


class KvWriteArgs(ctypes.Structure):
    _fields_ = [
        ("k_src", _vp), ("v_src", _vp), ("src_tok_stride", _i64), ("tok_pos", _vp),
        ("rope_table", _vp), ("rope_rows", _i64), ("pages", _vp), ("n_pages", _i32),
        ("k_dst", _vp), ("v_dst", _vp), ("dst_rows", _i64), ("dst_layers", _i32), ("layer", _i32),
        ("n_kv_heads", _i32), ("head_dim", _i32), ("hd_pad", _i32),
    ]


class KvReadArgs(ctypes.Structure):
    _fields_ = [
        ("k_src", _vp), ("v_src", _vp), ("src_rows", _i64), ("src_layers", _i32), ("layer", _i32),
        ("tok_pos", _vp), ("rope_table", _vp), ("rope_rows", _i64), ("pages", _vp), ("n_pages", _i32),
        ("n_kv_heads", _i32), ("head_dim", _i32), ("hd_pad", _i32), ("k_dst", _vp), ("v_dst", _vp),
    ]


_ERRORS = {
    1: errors.ShapeError,
    2: errors.MaskError,
    3: errors.ConfigError,
    4: errors.ValidationError,
    5: errors.CompatibilityError,
}

_lib = None
_lock = threading.Lock()


def load_library(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p.name} is not built; run `python -m paper_2503_08640_b200.build_ext` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(str(p))
        for name in EXPORTED_SYMBOLS:
            getattr(lib, name)  # AttributeError if a declared symbol is missing
        lib.dbsa_last_error.restype = ctypes.c_char_p
        lib.dbsa_abi_version.restype = ctypes.c_int
        lib.dbsa_attention.argtypes = [ctypes.POINTER(AttnArgs), _vp]
        lib.dbsa_lse_merge.argtypes = [ctypes.POINTER(MergeArgs), _vp]
        lib.dbsa_kv_write.argtypes = [ctypes.POINTER(KvWriteArgs), _vp]
        lib.dbsa_kv_read.argtypes = [ctypes.POINTER(KvReadArgs), _vp]
        lib.dbsa_rope_table.argtypes = [_vp, _i64, _vp, _i32, _i64, _vp]
        lib.dbsa_rope_table_f16.argtypes = [_vp, _i64, _vp, _i32, _i64, _vp]
        lib.dbsa_topk_select.argtypes = [_vp, _i64, _i64, _i64, _i32, _vp, _vp]
        lib.dbsa_rmsnorm.argtypes = [_vp, _vp, _vp, _i64, _i64, _f32, _vp]
        lib.dbsa_add_rmsnorm.argtypes = [_vp, _vp, _vp, _vp, _i64, _i64, _f32, _vp]
        lib.dbsa_silu_mul.argtypes = [_vp, _vp, _i64, _i64, _vp]
        lib.dbsa_label_logprob.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp]
        lib.dbsa_label_reduce.argtypes = [_vp, _vp, _i64, _i32, _vp, _vp, _vp]
        lib.dbsa_label_score.argtypes = [ctypes.POINTER(LabelScoreArgs), _vp]
        lib.dbsa_bm25_scores.argtypes = [_vp, _i64, _i32, _vp, _vp, _vp, _i64, ctypes.c_double, _vp, _vp]
        for name in EXPORTED_SYMBOLS[:-2]:
            getattr(lib, name).restype = ctypes.c_int
        if lib.dbsa_abi_version() != ABI_VERSION:
            raise errors.CompatibilityError(
                f"{p.name} ABI {lib.dbsa_abi_version()} != expected {ABI_VERSION}; rebuild"
            )
        if path is None:
            _lib = lib
        return lib


def check(code: int) -> None:
    if code == 0:
        return
    msg = (load_library().dbsa_last_error() or b"").decode("utf-8", "replace")
    raise _ERRORS.get(code, RuntimeError)(msg or f"libdbsa error {code}")


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())
