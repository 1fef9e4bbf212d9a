"""Retrieval around the hot path (reference: retrieval.py:1-388).

* `Bm25Index` keeps the reference's statistics and float64 scoring
  (retrieval.py:88-141, k1 = 1.2, b = 0.75).  `score_matrix` scores a batch of
  queries against every unit with numpy, adding each query term's float64
  contribution in query-term order -- the same IEEE operations in the same
  order as the reference's per-term loop, so scores are bit-identical.
* `select` / `order` reproduce retrieval.py:352-388 for one query on the host;
  `select_batch` is the GPU path: the score matrix goes to K4
  (dbsa_topk_select), which returns the anchor-first, ordered unit ids of
  every query, bit-exact with select + order.
* Grouping: the default random partition (retrieval.py:322-334, a Philox
  permutation chunked by block size).  The clustered strategies are one-time
  host setup outside the hot path; pass a precomputed
  partition to `pipeline.encode_pool` for those.
"""

from __future__ import annotations

import math
import re
from collections import Counter
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, ValidationError
from .kvstore import BLOCK_GRANULARITY, GRANULARITIES, SegmentRef, Selection

IN_ORDER, LOW_TO_HIGH, REVERSE = "in-order", "low-to-high", "reverse"
ORDERINGS = (IN_ORDER, LOW_TO_HIGH, REVERSE)
RANDOM, CLUSTERED, CLUSTERED_DIVERSE = "random", "clustered", "clustered-diverse"
GROUPINGS = (RANDOM, CLUSTERED, CLUSTERED_DIVERSE)
DEFAULT_K1, DEFAULT_B = 1.2, 0.75

_TERM = re.compile(r"[^\W_]+", re.UNICODE)


def bm25_tokenize(text: str) -> list[str]:
    """Lower-cased alphanumeric runs (retrieval.py:41-43)."""
    return _TERM.findall(text.lower())


@dataclass(frozen=True)
class GroupingStrategy:
    kind: str
    seed: int = 0
    swap_fraction: float = 0.10

    def __post_init__(self) -> None:
        if self.kind not in GROUPINGS:
            raise ValidationError(f"unknown grouping {self.kind!r}; expected one of {GROUPINGS}")
        if not 0.0 <= self.swap_fraction <= 1.0:
            raise ValidationError(f"swap_fraction must be in [0, 1], got {self.swap_fraction}")

    @classmethod
    def random(cls, seed: int = 0) -> "GroupingStrategy":
        return cls(RANDOM, seed)

    @classmethod
    def clustered(cls, seed: int = 0) -> "GroupingStrategy":
        return cls(CLUSTERED, seed)

    @classmethod
    def clustered_diverse(cls, seed: int = 0, swap_fraction: float = 0.10) -> "GroupingStrategy":
        return cls(CLUSTERED_DIVERSE, seed, swap_fraction)


@dataclass(frozen=True)
class BlockPartition:
    blocks: tuple[tuple[int, ...], ...]

    @property
    def n_blocks(self) -> int:
        return len(self.blocks)

    def n_examples(self) -> int:
        return sum(len(b) for b in self.blocks)

    def block_of(self) -> dict[int, int]:
        return {e: b for b, m in enumerate(self.blocks) for e in m}


def group(texts: list[str], block_size: int, strategy: GroupingStrategy) -> BlockPartition:
    """Random grouping (retrieval.py:322-334)."""
    n = len(texts)
    if n == 0:
        raise ValidationError("cannot group an empty pool")
    if block_size < 1:
        raise ValidationError(f"block_size must be >= 1, got {block_size}")
    if n < block_size:
        raise ValidationError(f"pool of {n} examples is smaller than block_size {block_size}")
    if strategy.kind != RANDOM:
        raise ConfigError(f"grouping {strategy.kind!r} is host setup outside the GPU path; "
                          "pass a precomputed BlockPartition to encode_pool(partition=...)")
    perm = np.random.Generator(np.random.Philox(int(strategy.seed))).permutation(n)
    return BlockPartition(tuple(tuple(int(x) for x in perm[i:i + block_size]) for i in range(0, n, block_size)))


class Bm25Index:
    """BM25 statistics plus unit metadata (retrieval.py:88-127)."""

    def __init__(self, texts, granularity, unit_refs, unit_examples, k1: float = DEFAULT_K1, b: float = DEFAULT_B):
        if granularity not in GRANULARITIES:
            raise ValidationError(f"unknown granularity {granularity!r}")
        if not (len(texts) == len(unit_refs) == len(unit_examples)):
            raise ValidationError("texts, unit_refs and unit_examples must align")
        if not texts:
            raise ValidationError("index needs at least one unit")
        self.granularity = granularity
        self.k1, self.b = float(k1), float(b)
        self.unit_refs = [tuple(r) for r in unit_refs]
        self.unit_examples = [tuple(e) for e in unit_examples]
        self.doc_terms = [Counter(bm25_tokenize(t)) for t in texts]
        self._finish()

    def _finish(self) -> None:
        self.doc_lens = [sum(c.values()) for c in self.doc_terms]
        self.n_docs = len(self.doc_terms)
        self.avgdl = sum(self.doc_lens) / self.n_docs
        self.df = Counter(t for c in self.doc_terms for t in c)
        self._dense = None

    def idf(self, term: str) -> float:
        d = self.df.get(term, 0)
        return math.log(1.0 + (self.n_docs - d + 0.5) / (d + 0.5))

    def _norms(self) -> np.ndarray:
        # k1 * (1 - b + b * dl / avgdl), per unit, same association as retrieval.py:134
        return np.array([self.k1 * (1.0 - self.b + self.b * dl / self.avgdl) for dl in self.doc_lens], np.float64)

    def score(self, query_terms: list[str], doc_id: int) -> float:
        if not 0 <= doc_id < self.n_docs:
            raise ValidationError(f"doc id {doc_id} outside index of {self.n_docs}")
        return float(self.score_matrix([query_terms])[0, doc_id])

    def _term_rows(self):
        """Per-term float64 contribution rows over all units, built lazily."""
        if self._dense is None:
            self._dense = ({}, self._norms())
        return self._dense

    def contribution(self, term: str) -> np.ndarray | None:
        rows, norm = self._term_rows()
        if term not in rows:
            if term not in self.df:
                rows[term] = None
            else:
                f = np.array([c.get(term, 0) for c in self.doc_terms], np.float64)
                idf = self.idf(term)
                with np.errstate(invalid="ignore", divide="ignore"):
                    r = idf * f * (self.k1 + 1.0) / (f + norm)
                rows[term] = np.where(f > 0, r, 0.0)
        return rows[term]

    def score_matrix(self, queries_terms) -> np.ndarray:
        """float64 [n_queries, n_units]; per query, the terms' contributions are
        added in query order (bit-exact with Bm25Index.score)."""
        out = np.zeros((len(queries_terms), self.n_docs), np.float64)
        for qi, terms in enumerate(queries_terms):
            acc = out[qi]
            for t in terms:
                r = self.contribution(t)
                if r is not None:
                    acc += r
        return out

    def device_tables(self, device=None):
        """(vocab {term: id}, tf uint16 [V, U], idf f64 [V], norm f64 [U]) on the
        GPU, built once; idf and norm are computed on the host with the
        reference's exact expressions (retrieval.py:125-134)."""
        from .engine import default_device

        dev = default_device(device)
        key = str(dev)
        cache = getattr(self, "_device_tables", None)
        if cache is None:
            cache = self._device_tables = {}
        if key not in cache:
            import torch

            vocab = {t: i for i, t in enumerate(sorted(self.df))}
            tf = np.zeros((max(1, len(vocab)), self.n_docs), np.uint16)
            for u, counter in enumerate(self.doc_terms):
                for t, f in counter.items():
                    if f > 65535:
                        raise ValidationError("term frequency above 65535 is not supported by the GPU BM25")
                    tf[vocab[t], u] = f
            idf = np.array([self.idf(t) for t in sorted(self.df)] or [0.0], np.float64)
            cache[key] = (vocab, torch.from_numpy(tf).to(dev), torch.from_numpy(idf).to(dev),
                          torch.from_numpy(self._norms()).to(dev))
        return cache[key]

    def score_matrix_device(self, queries_terms, device=None):
        """GPU BM25 (csrc/bm25.cu): float64 [n_queries, n_units] on the device,
        bit-identical to score_matrix."""
        import torch

        from . import ops

        vocab, tf, idf, norm = self.device_tables(device)
        width = max(1, max((len(t) for t in queries_terms), default=1))
        ids = np.full((len(queries_terms), width), -1, np.int32)
        for qi, terms in enumerate(queries_terms):
            for i, t in enumerate(terms):
                ids[qi, i] = vocab.get(t, -1)
        return ops.bm25_scores(torch.from_numpy(ids).to(tf.device), tf, idf, norm, self.k1 + 1.0)

    def to_json(self) -> dict:
        return {"granularity": self.granularity, "k1": self.k1, "b": self.b,
                "unit_refs": [list(r) for r in self.unit_refs], "unit_examples": [list(e) for e in self.unit_examples],
                "doc_terms": [dict(c) for c in self.doc_terms]}

    @classmethod
    def from_json(cls, data: dict) -> "Bm25Index":
        ix = cls.__new__(cls)
        ix.granularity = data["granularity"]
        ix.k1, ix.b = float(data["k1"]), float(data["b"])
        ix.unit_refs = [tuple(r) for r in data["unit_refs"]]
        ix.unit_examples = [tuple(e) for e in data["unit_examples"]]
        ix.doc_terms = [Counter(c) for c in data["doc_terms"]]
        ix._finish()
        return ix


def bm25_score(index: Bm25Index, query_terms: list[str], doc_id: int) -> float:
    return index.score(query_terms, doc_id)


def budget_for(ratio: float, n_units: int) -> int:
    """ceil(ratio * n) in float64 -- the reference's exact expression (retrieval.py:367)."""
    if not 0.0 < ratio <= 1.0:
        raise ValidationError(f"ratio must be in (0, 1], got {ratio}")
    return math.ceil(ratio * n_units)


def _check_gran(index: Bm25Index, granularity):
    if granularity is not None and granularity != index.granularity:
        raise ValidationError(f"index granularity {index.granularity!r} does not match requested {granularity!r}")


def _selection(index: Bm25Index, ids, scores) -> Selection:
    return Selection(index.granularity,
                     tuple(SegmentRef(int(u), *index.unit_refs[int(u)], score=float(scores[int(u)])) for u in ids))


def select(index: Bm25Index, query_text: str, ratio: float, granularity: str | None = None) -> Selection:
    """Anchor 0 plus the best budget-1 units by (-score, id) (retrieval.py:352-374)."""
    budget = budget_for(ratio, index.n_docs)
    _check_gran(index, granularity)
    scores = index.score_matrix([bm25_tokenize(query_text)])[0]
    rest = np.lexsort((np.arange(1, index.n_docs), -scores[1:]))[: budget - 1] + 1
    return _selection(index, [0, *rest.tolist()], scores)


def order(selection: Selection, strategy: str) -> Selection:
    """Anchor pinned; in-order / low-to-high / reverse (retrieval.py:377-388)."""
    if strategy not in ORDERINGS:
        raise ValidationError(f"unknown ordering {strategy!r}; expected one of {ORDERINGS}")
    head, rest = selection.units[0], list(selection.units[1:])
    key = {IN_ORDER: lambda u: u.unit_id, LOW_TO_HIGH: lambda u: (u.score, u.unit_id),
           REVERSE: lambda u: -u.unit_id}[strategy]
    return Selection(selection.granularity, (head, *sorted(rest, key=key)))


def select_batch(index: Bm25Index, query_texts, ratio: float, ordering: str, device=None, scores=None):
    """GPU selection for a batch: BM25 matrix (host, float64) -> K4 on device.
    Returns (int32 device tensor [n_queries, budget] of ordered unit ids,
    float64 host score matrix)."""
    import torch

    from . import ops
    from .engine import default_device

    if ordering not in ORDERINGS:
        raise ValidationError(f"unknown ordering {ordering!r}; expected one of {ORDERINGS}")
    budget = budget_for(ratio, index.n_docs)
    if scores is None:
        scores = index.score_matrix([bm25_tokenize(q) for q in query_texts])
    dev = default_device(device)
    ids = ops.topk_select(torch.from_numpy(scores).to(dev), budget, ordering)
    return ids, scores
