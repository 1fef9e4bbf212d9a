"""Decoder model surface of the drop-in API (reference: model.py:1-515).

Host-side types keep the reference's names, fields and validation:
`ModelConfig`, `ModelWeights` (float32 numpy tensors in the reference's
`x @ W` (in, out) layout), `init_random` (same Philox stream, so weights are
bit-identical to the reference's), `TokenSequence`, `ContextKV`, the rotary
helpers, and `forward_encode` / `forward_query` / `score_label`.

The forward passes themselves run on the GPU (engine.py): the weights are
uploaded once to a `DeviceModel` (bf16 GEMM operands, fp32 norms / embedding /
residual stream) and every attention call is the sm_100a kernel of
csrc/attn_sm100.cu.  There is no numpy compute path.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from .errors import CompatibilityError, ConfigError, MaskError, ShapeError, ValidationError

DTYPE = np.float32


@dataclass(frozen=True)
class ModelConfig:
    """Same fields, defaults and checks as model.py:35-100."""

    d_model: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab_size: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    max_seq_len: int = 32768

    def __post_init__(self) -> None:
        for name in ("d_model", "n_layers", "n_heads", "n_kv_heads", "head_dim", "ffn_dim", "vocab_size",
                     "max_seq_len"):
            if int(getattr(self, name)) <= 0:
                raise ConfigError(f"{name} must be positive, got {getattr(self, name)}")
        if self.rope_theta <= 0 or self.norm_eps <= 0:
            raise ConfigError("rope_theta and norm_eps must be positive")
        if self.n_heads % self.n_kv_heads:
            raise ConfigError(f"n_heads ({self.n_heads}) must be a multiple of n_kv_heads ({self.n_kv_heads})")
        if self.d_model != self.n_heads * self.head_dim:
            raise ConfigError(f"d_model ({self.d_model}) must equal n_heads*head_dim "
                              f"({self.n_heads}*{self.head_dim})")
        if self.head_dim % 2:
            raise ConfigError(f"head_dim must be even for rotary embeddings, got {self.head_dim}")

    @property
    def group_size(self) -> int:
        return self.n_heads // self.n_kv_heads

    def to_dict(self) -> dict:
        keys = ("d_model", "n_layers", "n_heads", "n_kv_heads", "head_dim", "ffn_dim", "vocab_size",
                "rope_theta", "norm_eps", "max_seq_len")
        return {k: getattr(self, k) for k in keys}

    @classmethod
    def from_dict(cls, data: dict) -> "ModelConfig":
        return cls(**data)

    def hash_bytes(self) -> bytes:
        """sha256 of the canonical JSON -- identical to the reference's, so
        config-compatibility checks agree across the two packages."""
        blob = json.dumps(self.to_dict(), sort_keys=True, separators=(",", ":"))
        return hashlib.sha256(blob.encode("utf-8")).digest()


def weight_shapes(config: ModelConfig) -> dict[str, tuple[int, ...]]:
    c = config
    qw, kw = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
    shapes = {"tok_embed": (c.vocab_size, c.d_model), "out_norm": (c.d_model,), "lm_head": (c.d_model, c.vocab_size)}
    for i in range(c.n_layers):
        p = f"layers.{i}."
        shapes.update({p + "attn_norm": (c.d_model,), p + "wq": (c.d_model, qw), p + "wk": (c.d_model, kw),
                       p + "wv": (c.d_model, kw), p + "wo": (qw, c.d_model), p + "ffn_norm": (c.d_model,),
                       p + "w_gate": (c.d_model, c.ffn_dim), p + "w_up": (c.d_model, c.ffn_dim),
                       p + "w_down": (c.ffn_dim, c.d_model)})
    return shapes


@dataclass
class ModelWeights:
    """Host weights (model.py:129-156).  `device()` uploads them once."""

    config: ModelConfig
    tensors: dict[str, np.ndarray]

    def __post_init__(self) -> None:
        want = weight_shapes(self.config)
        if set(self.tensors) != set(want):
            raise ShapeError(f"weight names mismatch: missing={sorted(set(want) - set(self.tensors))} "
                             f"extra={sorted(set(self.tensors) - set(want))}")
        for name, shape in want.items():
            t = self.tensors[name]
            if t.shape != shape:
                raise ShapeError(f"tensor {name}: expected shape {shape}, got {t.shape}")
            if t.dtype != DTYPE:
                self.tensors[name] = t.astype(DTYPE)
        self._device_models: dict = {}

    @property
    def config_hash(self) -> bytes:
        return self.config.hash_bytes()

    def checksum(self) -> str:
        h = hashlib.sha256()
        for name in sorted(self.tensors):
            h.update(name.encode("utf-8"))
            h.update(self.tensors[name].tobytes())
        return h.hexdigest()

    def device(self, device=None):
        """The GPU copy (cached per device)."""
        from .engine import DeviceModel, default_device

        dev = default_device(device)
        key = str(dev)
        if key not in self._device_models:
            self._device_models[key] = DeviceModel.from_weights(self, dev)
        return self._device_models[key]


def init_random(config: ModelConfig, seed: int) -> ModelWeights:
    """Scaled-uniform init from one Philox stream in sorted-name order
    (model.py:159-171): norms 1, embedding U(+-0.1), others U(+-1/sqrt(fan_in))."""
    rng = np.random.Generator(np.random.Philox(int(seed)))
    out: dict[str, np.ndarray] = {}
    for name, shape in sorted(weight_shapes(config).items()):
        if name.endswith("norm"):
            out[name] = np.ones(shape, DTYPE)
            continue
        bound = 0.1 if name == "tok_embed" else 1.0 / np.sqrt(shape[0])
        out[name] = rng.uniform(-bound, bound, size=shape).astype(DTYPE)
    return ModelWeights(config, out)


@dataclass(frozen=True)
class TokenSequence:
    """Token ids with strictly increasing non-negative positions (model.py:174-201)."""

    ids: tuple[int, ...]
    positions: tuple[int, ...]

    def __post_init__(self) -> None:
        if len(self.ids) != len(self.positions):
            raise ValidationError(f"ids ({len(self.ids)}) and positions ({len(self.positions)}) differ in length")
        if not self.ids:
            raise ValidationError("token sequence must be non-empty")
        p = np.asarray(self.positions, dtype=np.int64)
        if (p < 0).any():
            raise ValidationError("positions must be non-negative")
        if (np.diff(p) <= 0).any():
            raise ValidationError("positions must be strictly increasing")

    @classmethod
    def at_offset(cls, ids: Sequence[int], start: int) -> "TokenSequence":
        ids = tuple(int(i) for i in ids)
        return cls(ids, tuple(range(int(start), int(start) + len(ids))))

    def __len__(self) -> int:
        return len(self.ids)


# ----------------------------------------------------------------- rotary (host form)
def rope_angles(positions, head_dim: int, theta: float):
    """cos/sin of pos * theta^(-2i/hd), formed in float64 (model.py:205-209).
    The device table (ops.rope_table) is built from the same float64 angles."""
    freqs = theta ** (-np.arange(0, head_dim, 2, dtype=np.float64) / head_dim)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * freqs[None, :]
    return np.cos(ang), np.sin(ang)


def rope_rotate_heads(x, positions, theta: float) -> np.ndarray:
    """Rotate (T, heads, hd) at per-token positions, paired halves (model.py:222-239)."""
    x = np.asarray(x, dtype=DTYPE)
    if x.ndim != 3:
        raise ShapeError(f"rope_rotate_heads expects (T, heads, head_dim), got {x.shape}")
    hd = x.shape[-1]
    if hd % 2:
        raise ConfigError(f"head_dim must be even for rotary embeddings, got {hd}")
    c, s = rope_angles(positions, hd, theta)
    c, s = c[:, None, :], s[:, None, :]
    a, b = x[..., : hd // 2].astype(np.float64), x[..., hd // 2:].astype(np.float64)
    return np.concatenate([a * c - b * s, a * s + b * c], axis=-1).astype(DTYPE)


def rope_rotate(vec, position: int, theta: float) -> np.ndarray:
    vec = np.asarray(vec, dtype=DTYPE)
    if vec.ndim != 1:
        raise ShapeError(f"rope_rotate expects a 1-D vector, got shape {vec.shape}")
    if vec.shape[0] % 2:
        raise ConfigError(f"head_dim must be even for rotary embeddings, got {vec.shape[0]}")
    return rope_rotate_heads(vec[None, None, :], np.array([position]), theta)[0, 0]


LayerKV = tuple  # (keys, values), each (T, n_kv_heads, head_dim)


@dataclass
class ContextKV:
    """Rotated per-layer context for forward_encode (model.py:245-264)."""

    positions: np.ndarray
    layers: list = field(default_factory=list)

    @classmethod
    def empty(cls, config: ModelConfig) -> "ContextKV":
        z = np.zeros((0, config.n_kv_heads, config.head_dim), DTYPE)
        return cls(np.zeros(0, np.int64), [(z, z) for _ in range(config.n_layers)])

    def __len__(self) -> int:
        return int(np.asarray(self.positions).shape[0])


def _check_ids(config: ModelConfig, ids, positions) -> None:
    ids = np.asarray(ids, dtype=np.int64)
    if ids.min() < 0 or ids.max() >= config.vocab_size:
        raise ValidationError(f"token id outside vocabulary [0, {config.vocab_size})")
    if int(np.max(positions)) >= config.max_seq_len:
        raise ValidationError(f"position {int(np.max(positions))} exceeds max_seq_len {config.max_seq_len}")


def _weights_of(weights):
    """ModelWeights -> its DeviceModel; a DeviceModel passes through."""
    from .engine import DeviceModel

    return weights if isinstance(weights, DeviceModel) else weights.device()


def forward_encode(weights, tokens: TokenSequence, context: ContextKV | None, token_mask):
    """Encode one group against an explicit rotated context (model.py:363-378).

    Returns (per-layer pre-rotation (K, V) float32, final hidden float32).  The
    token mask must have the block structure the sparse kernel implements --
    context columns all visible, self part causal -- which is the only form
    the reference pipeline produces (masks.block_mask_rows, masks.py:164-177);
    any other mask raises MaskError (this path has no dense fallback).
    """
    from . import engine

    dm = _weights_of(weights)
    cfg = dm.config
    if context is None:
        context = ContextKV.empty(cfg)
    if len(context.layers) != cfg.n_layers:
        raise ShapeError(f"context has {len(context.layers)} layers, model has {cfg.n_layers}")
    n_ctx, t = len(context), len(tokens)
    for k, v in context.layers:
        want = (n_ctx, cfg.n_kv_heads, cfg.head_dim)
        if k.shape != want or v.shape != want:
            raise ShapeError(f"context KV shape {k.shape}/{v.shape}, expected {want}")
    _check_ids(cfg, tokens.ids, tokens.positions)
    if n_ctx and int(np.max(context.positions)) >= int(tokens.positions[0]):
        raise ValidationError("context positions overlap new token positions "
                              f"(context max {int(np.max(context.positions))}, new min {tokens.positions[0]})")
    mask = np.asarray(token_mask, dtype=bool)
    if mask.shape != (t, n_ctx + t):
        raise MaskError(f"token mask shape {mask.shape}, expected {(t, n_ctx + t)}")
    if not mask.any(axis=1).all():
        raise MaskError("fully-masked query row in token mask")
    if not (mask[:, :n_ctx].all() and np.array_equal(mask[:, n_ctx:], np.tri(t, dtype=bool))):
        raise MaskError("the sm_100a kernel implements [context all | self causal] token masks only")
    return engine.forward_explicit_context(dm, tokens, context)


def logits_from_hidden(weights, hidden) -> np.ndarray:
    from . import engine

    return engine.logits_host(_weights_of(weights), hidden)


def _assembled_for(dm, assembled):
    if assembled is None:
        return None
    if assembled.config_hash != dm.config.hash_bytes():
        raise CompatibilityError("assembled cache was built for a different model config")
    return assembled


def forward_query(weights, assembled, query: TokenSequence) -> np.ndarray:
    """Logits of every query position against an assembled selection, full
    attention to it and causal within the query (model.py:400-411)."""
    from . import engine

    dm = _weights_of(weights)
    asm = _assembled_for(dm, assembled)
    n_ctx = asm.total_tokens if asm is not None else 0
    if query.positions[0] != n_ctx:
        raise ValidationError(f"query positions must start at the assembled length {n_ctx}, got {query.positions[0]}")
    _check_ids(dm.config, query.ids, query.positions)
    return engine.forward_query(dm, asm, list(query.ids))


def log_softmax_rows(logits) -> np.ndarray:
    x = np.asarray(logits, dtype=np.float64)
    x = x - x.max(axis=1, keepdims=True)
    return x - np.log(np.exp(x).sum(axis=1, keepdims=True))


def score_label(weights, assembled, query_ids: Sequence[int], label_ids: Sequence[int]) -> float:
    """Teacher-forced sum of label-token log-probs (model.py:420-443)."""
    from . import engine

    q, lab = [int(i) for i in query_ids], [int(i) for i in label_ids]
    if not lab:
        raise ValidationError("label must be non-empty")
    if not q:
        raise ValidationError("query must be non-empty")
    dm = _weights_of(weights)
    vocab = dm.config.vocab_size
    if any(not 0 <= tok < vocab for tok in q + lab):
        raise ValidationError(f"token id outside vocabulary [0, {vocab})")
    asm = _assembled_for(dm, assembled)
    n_ctx = asm.total_tokens if asm is not None else 0
    if n_ctx + len(q) + len(lab) > dm.config.max_seq_len:
        raise ValidationError(f"position {n_ctx + len(q) + len(lab) - 1} exceeds max_seq_len {dm.config.max_seq_len}")
    return float(engine.score_labels(dm, asm, q, [lab])[0])
