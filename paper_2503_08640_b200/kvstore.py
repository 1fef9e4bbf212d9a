"""Group KV cache in HBM pages (component K2; reference: kvstore.py:1-235).

Reference layout: per layer, per group, a float32 numpy array of PRE-rotation
keys and one of values; stage 2 `assemble` concatenates the selected spans and
rotates the keys at new positions 0..T'-1 -- a per-query copy of ~3.5 GB at
the Llama-3.1-8B / 90k / 30% configuration.

Here one page store per cache holds every group (engine.PageStore):

    K   [L][Hkv][rows][HDP]  bf16, keys ROTATED at their original positions
    V^T [L][Hkv][HDP][rows]  bf16, values transposed (token axis contiguous)

A group owns a contiguous run of whole 64-token pages (pages never span
groups), so a selected unit -- a whole group or a demonstration's token span
inside one -- is the row range (row0 + start, end - start) of that group.
`assemble` therefore copies nothing: it returns the ordered chunk table
(row, length, delta = new_start - original_start) and K3 applies the
re-positioning on the QUERY side, R(p_q - delta) q . R(p_orig) k ==
R(p_q) q . R(p_new) k.  The reference's array views (`segment`,
`AssembledCache.layers`) are still provided, materialised on demand from the
pages for API users and tests.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import model
from .errors import CompatibilityError, FormatError, ShapeError, ValidationError

CACHE_MAGIC = b"DBSACACH"  # on-disk format of kvstore.py:238-316
CACHE_VERSION = 1

BLOCK_GRANULARITY = "block"
EXAMPLE_GRANULARITY = "example"
GRANULARITIES = (BLOCK_GRANULARITY, EXAMPLE_GRANULARITY)


@dataclass(frozen=True)
class BlockEntry:
    """kvstore.py:26-33 plus the group's first page row in the store."""

    block_id: int
    token_count: int
    pos_start: int
    pos_end: int
    text_digest: bytes
    example_spans: tuple[tuple[int, int], ...]
    row0: int = 0


def _check_spans(spans, token_count):
    spans = tuple((int(a), int(b)) for a, b in spans)
    for a, b in spans:
        if not 0 <= a < b <= token_count:
            raise ValidationError(f"example span ({a}, {b}) outside block of {token_count}")
    return spans


class SegmentedKVCache:
    """Append-only group cache backed by HBM pages (kvstore.py:36-106).

    Single writer while building; `seal()` freezes it for concurrent
    read-only use by stage-2 workers.
    """

    def __init__(self, config: model.ModelConfig, device=None, capacity_tokens: int = 0):
        from .engine import PageStore, default_device

        self.config = config
        self.config_hash = config.hash_bytes()
        self.blocks: list[BlockEntry] = []
        self.sealed = False
        self.store = PageStore(config, default_device(device), capacity_tokens)

    @property
    def n_blocks(self) -> int:
        return len(self.blocks)

    @property
    def total_tokens(self) -> int:
        return self.blocks[-1].pos_end if self.blocks else 0

    @property
    def device(self):
        return self.store.device

    def seal(self) -> "SegmentedKVCache":
        self.sealed = True
        return self

    # ---- allocation (used by encode_blocks, which writes the pages on the GPU)
    def _reserve(self, counts, digests, spans_list) -> list[BlockEntry]:
        if self.sealed:
            raise ValidationError("cache is sealed; cannot append")
        new = []
        start = self.total_tokens
        rows = self.store.reserve([int(c) for c in counts])
        for i, (n, dg, sp) in enumerate(zip(counts, digests, spans_list)):
            n = int(n)
            if n <= 0:
                raise ShapeError("block token counts must be positive")
            if len(dg) != 32:
                raise ValidationError("text digest must be 32 bytes (SHA-256)")
            new.append(BlockEntry(self.n_blocks + i, n, start, start + n, bytes(dg), _check_spans(sp, n), rows[i]))
            start += n
        self.blocks.extend(new)
        return new

    def _reserve_subset(self, counts, digests, spans_list, present) -> list[BlockEntry]:
        """Metadata for every group, pages only for the groups in `present`
        (a group-sharded cache, parallel.py); absent groups get row0 = -1."""
        if self.sealed or self.blocks:
            raise ValidationError("a sharded cache is reserved once, empty")
        present = set(int(g) for g in present)
        rows = iter(self.store.reserve([int(counts[g]) for g in sorted(present)]))
        row_of = {g: next(rows) for g in sorted(present)}
        start = 0
        for g, (n, dg, sp) in enumerate(zip(counts, digests, spans_list)):
            n = int(n)
            self.blocks.append(BlockEntry(g, n, start, start + n, bytes(dg), _check_spans(sp, n), row_of.get(g, -1)))
            start += n
        return self.blocks

    def append_block(self, block_id: int, pre_rotation_kv, text_digest: bytes,
                     example_spans: tuple[tuple[int, int], ...] = ()) -> "SegmentedKVCache":
        """Append one group's host pre-rotation K/V (kvstore.py:70-106): the
        K2w kernel rotates K at the group's original positions into its pages."""
        if self.sealed:
            raise ValidationError("cache is sealed; cannot append")
        if block_id != self.n_blocks:
            raise ValidationError(f"block ids must be appended in order: expected {self.n_blocks}, got {block_id}")
        if len(pre_rotation_kv) != self.config.n_layers:
            raise ShapeError(f"expected KV for {self.config.n_layers} layers, got {len(pre_rotation_kv)}")
        n = int(np.asarray(pre_rotation_kv[0][0]).shape[0])
        want = (n, self.config.n_kv_heads, self.config.head_dim)
        for k, v in pre_rotation_kv:
            if np.asarray(k).shape != want or np.asarray(v).shape != want:
                raise ShapeError(f"KV segment shape {np.asarray(k).shape}/{np.asarray(v).shape}, expected {want}")
        if len(text_digest) != 32:
            raise ValidationError("text digest must be 32 bytes (SHA-256)")
        _check_spans(example_spans, n)
        (entry,) = self._reserve([n], [text_digest], [example_spans])
        self.store.write_host_group(entry, pre_rotation_kv)
        return self

    def segment(self, layer: int, block_id: int):
        """(pre-rotation K, V) float32 (T, Hkv, hd) of one group, read back from
        the pages and un-rotated on the host (cold path)."""
        e = self.blocks[block_id]
        if e.row0 < 0:
            raise ValidationError(f"group {block_id} is held by another shard")
        k_rot, v = self.store.read_rows(layer, e.row0, e.token_count)
        pos = np.arange(e.pos_start, e.pos_end, dtype=np.int64)
        return model.rope_rotate_heads(k_rot, -pos, self.config.rope_theta), v


@dataclass(frozen=True)
class SegmentRef:
    """One selectable unit: a whole group or a demonstration span (kvstore.py:109-121)."""

    unit_id: int
    block_id: int
    start: int
    end: int
    score: float = 0.0

    def length(self) -> int:
        return self.end - self.start


@dataclass(frozen=True)
class Selection:
    """Ordered units, anchor first, distinct ids (kvstore.py:124-147)."""

    granularity: str
    units: tuple[SegmentRef, ...]

    def __post_init__(self) -> None:
        if self.granularity not in GRANULARITIES:
            raise ValidationError(f"unknown granularity {self.granularity!r}")
        if not self.units:
            raise ValidationError("selection must be non-empty")
        ids = [u.unit_id for u in self.units]
        if len(set(ids)) != len(ids):
            raise ValidationError("selection unit ids must be distinct")
        if self.units[0].block_id != 0 or self.units[0].start != 0:
            raise ValidationError("selection must start with the anchor block segment")

    @property
    def unit_ids(self) -> tuple[int, ...]:
        return tuple(u.unit_id for u in self.units)

    def total_tokens(self) -> int:
        return sum(u.length() for u in self.units)


def all_blocks_selection(cache: SegmentedKVCache) -> Selection:
    return Selection(BLOCK_GRANULARITY,
                     tuple(SegmentRef(e.block_id, e.block_id, 0, e.token_count) for e in cache.blocks))


class AssembledCache:
    """A selection re-positioned to 0..T'-1 (kvstore.py:157-185).

    `chunks` is what K3 consumes: int64 rows of (pool row, n_tok, delta).
    `layers` (rotated K, V per layer, float32) is materialised lazily from the
    pages, only when an API caller asks for it.
    """

    def __init__(self, config_hash: bytes, total_tokens: int, provenance_blocks, provenance_offsets,
                 selection: Selection | None = None, cache: SegmentedKVCache | None = None, chunks=None,
                 layers=None):
        self.config_hash = config_hash
        self.total_tokens = int(total_tokens)
        self.provenance_blocks = provenance_blocks
        self.provenance_offsets = provenance_offsets
        self.selection = selection
        self.cache = cache
        self.chunks = np.zeros((0, 3), np.int64) if chunks is None else chunks
        self._layers = layers

    @classmethod
    def empty(cls, config: model.ModelConfig) -> "AssembledCache":
        z = np.zeros((0, config.n_kv_heads, config.head_dim), np.float32)
        return cls(config.hash_bytes(), 0, np.zeros(0, np.int64), np.zeros(0, np.int64),
                   layers=tuple((z, z) for _ in range(config.n_layers)))

    @property
    def layers(self):
        if self._layers is None:
            c = self.cache.config
            pos = np.arange(self.total_tokens, dtype=np.int64)
            out = []
            for layer in range(c.n_layers):
                parts = [self.cache.segment(layer, u.block_id) for u in self.selection.units]
                k = np.concatenate([p[0][u.start:u.end] for p, u in zip(parts, self.selection.units)])
                v = np.concatenate([p[1][u.start:u.end] for p, u in zip(parts, self.selection.units)])
                out.append((model.rope_rotate_heads(k, pos, c.rope_theta), v))
            self._layers = tuple(out)
        return self._layers

    def provenance(self, position: int) -> tuple[int, int]:
        return int(self.provenance_blocks[position]), int(self.provenance_offsets[position])


def chunk_table(cache: SegmentedKVCache, units) -> np.ndarray:
    """(row, n_tok, delta) per unit in order; delta = new start - original start."""
    rows = np.empty((len(units), 3), np.int64)
    new_start = 0
    for i, u in enumerate(units):
        e = cache.blocks[u.block_id]
        n = u.end - u.start
        rows[i] = (e.row0 + u.start, n, new_start - (e.pos_start + u.start))
        new_start += n
    return rows


def _validate_units(cache: SegmentedKVCache, units) -> None:
    for u in units:
        if not 0 <= u.block_id < cache.n_blocks:
            raise ValidationError(f"unknown block id {u.block_id}")
        n = cache.blocks[u.block_id].token_count
        if not 0 <= u.start < u.end <= n:
            raise ValidationError(f"segment span ({u.start}, {u.end}) outside block {u.block_id} of {n} tokens")


def assemble(cache: SegmentedKVCache, selection: Selection) -> AssembledCache:
    """Re-position a selection to 0..T'-1 without moving any KV (kvstore.py:188-221)."""
    _validate_units(cache, selection.units)
    lens = [u.length() for u in selection.units]
    prov_b = np.repeat(np.array([u.block_id for u in selection.units], np.int64), lens)
    prov_o = np.concatenate([np.arange(u.start, u.end, dtype=np.int64) for u in selection.units])
    return AssembledCache(cache.config_hash, sum(lens), prov_b, prov_o, selection, cache,
                          chunk_table(cache, selection.units))


def storage_bytes(config: model.ModelConfig, n_tokens: int, bytes_per_value: int) -> int:
    """K + V bytes of n_tokens (kvstore.py:224-230)."""
    if n_tokens < 0:
        raise ValidationError(f"n_tokens must be non-negative, got {n_tokens}")
    if bytes_per_value not in (2, 4):
        raise ValidationError(f"bytes_per_value must be 2 or 4, got {bytes_per_value}")
    return 2 * config.n_layers * config.n_kv_heads * config.head_dim * bytes_per_value * n_tokens


def check_compatible(cache: SegmentedKVCache, config: model.ModelConfig) -> None:
    if cache.config_hash != config.hash_bytes():
        raise CompatibilityError("cache and weights were built for different configs")


# ------------------------------------------------------------------ cache files
# Byte-compatible with the reference's DBSACACH format (kvstore.py:238-316):
# header, block table, then per layer, per group, float32 pre-rotation K
# followed by V in [t, Hkv, hd] order.  Pages are read/written on the GPU: K2r
# un-rotates a whole layer of pages in one launch, and K2w writes a whole
# layer from the file in one launch.
def _header_bytes(cache) -> bytes:
    import struct

    cfg = cache.config
    out = [CACHE_MAGIC, struct.pack("<I", CACHE_VERSION), cache.config_hash,
           struct.pack("<III", cfg.n_layers, cfg.n_kv_heads, cfg.head_dim), struct.pack("<I", cache.n_blocks)]
    for e in cache.blocks:
        out.append(struct.pack("<IIQQ", e.block_id, e.token_count, e.pos_start, e.pos_end))
        out.append(e.text_digest)
        out.append(struct.pack("<I", len(e.example_spans)))
        out += [struct.pack("<II", a, b) for a, b in e.example_spans]
    return b"".join(out)


def serialize(cache: SegmentedKVCache, path) -> None:
    """Write the cache in the reference's file format (kvstore.py:238-258)."""
    import torch

    from . import engine, ops

    cfg = cache.config
    if any(e.row0 < 0 for e in cache.blocks):
        raise ValidationError("a group-sharded cache holds only part of the pool; serialize each owner's groups")
    store, dev = cache.store, cache.device
    total = cache.total_tokens
    if total == 0:  # an empty cache is a header with an empty block table (kvstore.py:238-258)
        with open(path, "wb") as fh:
            fh.write(_header_bytes(cache))
        return
    pos = torch.arange(total, dtype=torch.int32, device=dev)
    pages = engine._pages_for([(e.pos_start, e.token_count, e.row0) for e in cache.blocks])
    pdev = ops.to_device(pages, dev)
    k = torch.empty((total, cfg.n_kv_heads, cfg.head_dim), dtype=torch.float32, device=dev)
    v = torch.empty_like(k)
    with open(path, "wb") as fh:
        fh.write(_header_bytes(cache))
        for layer in range(cfg.n_layers):
            ops.kv_read(store.k, store.v, store.rows, cfg.n_layers, layer, pos, store.rope, pdev, len(pages),
                        cfg.n_kv_heads, cfg.head_dim, k, v)
            kh, vh = k.cpu().numpy(), v.cpu().numpy()
            for e in cache.blocks:
                fh.write(np.ascontiguousarray(kh[e.pos_start:e.pos_end], dtype="<f4").tobytes())
                fh.write(np.ascontiguousarray(vh[e.pos_start:e.pos_end], dtype="<f4").tobytes())


def deserialize(path, config: model.ModelConfig, device=None) -> SegmentedKVCache:
    """Read a reference-format cache file straight into HBM pages
    (kvstore.py:261-316): same validation and exceptions."""
    import struct

    import torch

    from . import engine, ops

    def read(fh, n: int, what: str) -> bytes:
        data = fh.read(n)
        if len(data) != n:
            raise FormatError(f"truncated cache file while reading {what}")
        return data

    with open(path, "rb") as fh:
        if read(fh, 8, "magic") != CACHE_MAGIC:
            raise FormatError("not a KV cache file (bad magic)")
        (version,) = struct.unpack("<I", read(fh, 4, "version"))
        if version != CACHE_VERSION:
            raise FormatError(f"unsupported cache file version {version}")
        if read(fh, 32, "config hash") != config.hash_bytes():
            raise CompatibilityError("cache file was built for a different model config")
        dims = struct.unpack("<III", read(fh, 12, "dims"))
        if dims != (config.n_layers, config.n_kv_heads, config.head_dim):
            raise CompatibilityError("cache dims disagree with model config")
        (n_blocks,) = struct.unpack("<I", read(fh, 4, "block count"))
        table = []
        for _ in range(n_blocks):
            bid, count, start, end = struct.unpack("<IIQQ", read(fh, 24, "block entry"))
            digest = read(fh, 32, "digest")
            (n_spans,) = struct.unpack("<I", read(fh, 4, "span count"))
            spans = tuple(struct.unpack("<II", read(fh, 8, "span")) for _ in range(n_spans))
            table.append((bid, count, start, end, digest, spans))
        expect_start = 0
        for i, (bid, count, start, end, _, _) in enumerate(table):
            if bid != i or start != expect_start or end != start + count or count <= 0:
                raise FormatError(f"inconsistent block table entry {i}")
            expect_start = end
        cache = SegmentedKVCache(config, device, capacity_tokens=expect_start)
        if expect_start == 0:  # empty cache: header only
            if fh.read(1):
                raise FormatError("trailing bytes after final segment")
            return cache.seal()
        entries = cache._reserve([t[1] for t in table], [t[4] for t in table], [t[5] for t in table])
        total, per_tok = expect_start, config.n_kv_heads * config.head_dim
        dev = cache.device
        pos = torch.arange(total, dtype=torch.int32, device=dev)
        pages = engine._pages_for([(e.pos_start, e.token_count, e.row0) for e in entries])
        pdev = ops.to_device(pages, dev)
        st = cache.store
        for layer in range(config.n_layers):
            kb = np.empty((total, per_tok), np.float32)
            vb = np.empty((total, per_tok), np.float32)
            for e in entries:
                n_vals = e.token_count * per_tok
                kb[e.pos_start:e.pos_end] = np.frombuffer(read(fh, 4 * n_vals, "keys"), "<f4").reshape(-1, per_tok)
                vb[e.pos_start:e.pos_end] = np.frombuffer(read(fh, 4 * n_vals, "values"), "<f4").reshape(-1, per_tok)
            kd = torch.from_numpy(kb).to(dev).to(torch.bfloat16)
            vd = torch.from_numpy(vb).to(dev).to(torch.bfloat16)
            ops.kv_write(kd, vd, per_tok, pos, st.rope, pdev, len(pages), st.k, st.v, st.rows, config.n_layers,
                         layer, config.n_kv_heads, config.head_dim)
        if fh.read(1):
            raise FormatError("trailing bytes after final segment")
    torch.cuda.current_stream(dev).synchronize()
    return cache.seal()


def expected_file_size(config: model.ModelConfig, token_counts, spans_per_block) -> int:
    """Bytes `serialize` writes (kvstore.py:319-324)."""
    header = 8 + 4 + 32 + 12 + 4
    table = sum(24 + 32 + 4 + 8 * len(s) if not isinstance(s, int) else 24 + 32 + 4 + 8 * s for s in spans_per_block)
    return header + table + 2 * config.n_layers * config.n_kv_heads * config.head_dim * 4 * sum(token_counts)
