"""Cache files in the reference's DBSACACH format (kvstore.py:238-324).

tests/golden/cache_tiny.dbsacache was written by the unmodified reference's
`serialize` (tests/golden/make_golden.py).  The CPU tests cover the header /
table parser and its error mapping.  The GPU tests check four things:
* deserialize into HBM pages (K2w) reads the reference's values;
* serialize from pages (K2r) writes the same header and table bytes;
* serialize writes the reference's values within bf16 tolerance;
* the file size matches expected_file_size.
"""

import json
import struct
from pathlib import Path

import numpy as np
import pytest

import paper_2503_08640_b200 as P
from paper_2503_08640_b200 import kvstore, tokenizer

GOLDEN = Path(__file__).resolve().parent / "golden"
KV_TOL = 3e-2


def _meta():
    return json.loads((GOLDEN / "cache_tiny.json").read_text())


def _cfg(meta):
    return P.ModelConfig(vocab_size=tokenizer.VOCAB_SIZE, **meta["model"])


def _parse(raw: bytes, cfg):
    """Independent numpy parse of a DBSACACH byte string -> (table bytes, entries, per-layer (k, v) lists)."""
    off = 8 + 4 + 32 + 12
    (n_blocks,) = struct.unpack_from("<I", raw, off)
    off += 4
    entries = []
    for _ in range(n_blocks):
        bid, count, start, end = struct.unpack_from("<IIQQ", raw, off)
        off += 24 + 32
        (ns,) = struct.unpack_from("<I", raw, off)
        off += 4 + 8 * ns
        entries.append((bid, count, start, end))
    head = raw[:off]
    per = cfg.n_kv_heads * cfg.head_dim
    layers = []
    for _ in range(cfg.n_layers):
        kv = []
        for _, count, _, _ in entries:
            n = count * per * 4
            k = np.frombuffer(raw[off:off + n], "<f4").reshape(count, cfg.n_kv_heads, cfg.head_dim)
            v = np.frombuffer(raw[off + n:off + 2 * n], "<f4").reshape(count, cfg.n_kv_heads, cfg.head_dim)
            kv.append((k, v))
            off += 2 * n
        layers.append(kv)
    assert off == len(raw)
    return head, entries, layers


def test_reference_file_layout_and_size():
    meta = _meta()
    cfg = _cfg(meta)
    raw = (GOLDEN / "cache_tiny.dbsacache").read_bytes()
    assert raw[:8] == kvstore.CACHE_MAGIC and len(raw) == meta["file_size"]
    _, entries, _ = _parse(raw, cfg)
    # example granularity: spans recorded, so the size formula needs the span counts
    off, spans = 8 + 4 + 32 + 12 + 4, []
    for _ in entries:
        off += 24 + 32
        (ns,) = struct.unpack_from("<I", raw, off)
        off += 4 + 8 * ns
        spans.append(ns)
    assert kvstore.expected_file_size(cfg, [e[1] for e in entries], spans) == len(raw)


@pytest.mark.parametrize("mutate,exc", [
    (lambda b: b"XXXXXXXX" + b[8:], P.FormatError),
    (lambda b: b[:8] + struct.pack("<I", 9) + b[12:], P.FormatError),
    (lambda b: b[:12] + bytes(32) + b[44:], P.CompatibilityError),
    (lambda b: b[:40], P.FormatError),
])
def test_reference_file_errors(tmp_path, mutate, exc):
    meta = _meta()
    raw = (GOLDEN / "cache_tiny.dbsacache").read_bytes()
    bad = tmp_path / "bad.dbsacache"
    bad.write_bytes(mutate(raw))
    with pytest.raises(exc):
        kvstore.deserialize(bad, _cfg(meta))


@pytest.mark.gpu
def test_deserialize_reference_file_into_pages_and_back(tmp_path):
    meta = _meta()
    cfg = _cfg(meta)
    raw = (GOLDEN / "cache_tiny.dbsacache").read_bytes()
    head, entries, layers = _parse(raw, cfg)
    cache = kvstore.deserialize(GOLDEN / "cache_tiny.dbsacache", cfg)
    assert cache.sealed and cache.n_blocks == meta["n_blocks"] and cache.total_tokens == meta["total_tokens"]
    worst = 0.0
    for layer in range(cfg.n_layers):
        for b in range(cache.n_blocks):
            k, v = cache.segment(layer, b)
            rk, rv = layers[layer][b]
            worst = max(worst, float(np.abs(k - rk).max()), float(np.abs(v - rv).max()))
    assert worst < KV_TOL, worst
    out = tmp_path / "ours.dbsacache"
    kvstore.serialize(cache, out)
    raw2 = out.read_bytes()
    assert len(raw2) == len(raw)
    head2, _, layers2 = _parse(raw2, cfg)
    assert head2 == head  # header + block table byte-identical
    worst = max(float(np.abs(a[0] - b[0]).max()) for la, lb in zip(layers, layers2) for a, b in zip(la, lb))
    assert worst < KV_TOL, worst
    # our file reads back: V exactly (bf16 -> f32 -> bf16), K up to the bf16
    # rounding of the un-rotate / re-rotate round trip
    cache2 = kvstore.deserialize(out, cfg)
    import torch

    n = cache.store.used_rows
    assert torch.equal(cache2.store.v[..., :n], cache.store.v[..., :n])
    dk = (cache2.store.k[:, :, :n].float() - cache.store.k[:, :, :n].float()).abs().max().item()
    assert dk < 2e-2, dk


@pytest.mark.gpu
def test_empty_cache_round_trip(tmp_path):
    """An empty cache (no groups) writes a header-only file and reads back as a
    sealed empty cache, as the reference's serialize/deserialize allow."""
    meta = _meta()
    cfg = _cfg(meta)
    cache = P.SegmentedKVCache(cfg).seal()
    out = tmp_path / "empty.dbsacache"
    kvstore.serialize(cache, out)
    raw = out.read_bytes()
    assert len(raw) == kvstore.expected_file_size(cfg, [], [])
    back = kvstore.deserialize(out, cfg)
    assert back.sealed and back.n_blocks == 0 and back.total_tokens == 0
