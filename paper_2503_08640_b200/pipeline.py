"""Stage-1 pre-encode and stage-2 retrieve-and-answer calls
(reference: pipeline.py:1-482).

Same names, signatures, validation and return types as the reference:
`encode_pool(weights, task, config) -> EncodedPool`,
`encode_blocks(weights, cache, new_blocks, pattern) -> int`,
`Runner(weights, cache, index, task, config).infer(query) -> (label, QueryMetrics)`
and `infer(...)`.  `weights` is the reference's host `ModelWeights` (uploaded
once) or an `engine.DeviceModel`.  Added for throughput: `Runner.infer_batch`
and the lower-level `Stage2Session`, which take many queries per forward and
select their groups with K4 on the device.

Methods: "dbsa" (the hot path), "fixed" (all groups of the cache, the
reference's cached-ICL baseline) and "zero" (no context) run on the same
kernels.  "ret" re-encodes retrieved text without a cache; it is a baseline
outside the DBSA hot path and is rejected with ConfigError.
"""

from __future__ import annotations

import hashlib
import threading
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import engine, kvstore, masks, retrieval, tokenizer
from .errors import CompatibilityError, ConfigError, ValidationError
from .metrics import Metrics, QueryMetrics, flops_attention

DBSA, FIXED_ICL, RET_ICL, ZERO_SHOT = "dbsa", "fixed", "ret", "zero"
METHODS = (DBSA, FIXED_ICL, RET_ICL, ZERO_SHOT)
_ALIASES = {"dbsa": DBSA, "fixed": FIXED_ICL, "fixed-icl": FIXED_ICL, "ret": RET_ICL, "ret-icl": RET_ICL,
            "reticl": RET_ICL, "zero": ZERO_SHOT, "zero-shot": ZERO_SHOT}


def canonical_method(name: str) -> str:
    try:
        return _ALIASES[name.lower()]
    except KeyError:
        raise ValidationError(f"unknown method {name!r}; expected one of {METHODS}") from None


@dataclass(frozen=True)
class Demonstration:
    query: str
    answer: str

    def __post_init__(self) -> None:
        if not self.query.strip() or not self.answer.strip():
            raise ValidationError("demonstration query and answer must be non-empty")

    def raw_text(self) -> str:
        return f"{self.query} {self.answer}"


@dataclass(frozen=True)
class PromptTemplate:
    """Rendering of demos / queries / labels (pipeline.py:58-71)."""

    demo_format: str = "Q: {query}\nA: {answer}\n\n"
    query_format: str = "Q: {query}\nA:"
    label_format: str = " {label}"

    def render_demo(self, demo: Demonstration) -> str:
        return self.demo_format.format(query=demo.query, answer=demo.answer)

    def render_query(self, query: str) -> str:
        return self.query_format.format(query=query)

    def render_label(self, label: str) -> str:
        return self.label_format.format(label=label)


@dataclass(frozen=True)
class TaskSpec:
    pool: tuple[Demonstration, ...]
    labels: tuple[str, ...]
    template: PromptTemplate = PromptTemplate()

    def __post_init__(self) -> None:
        if not self.pool:
            raise ValidationError("demonstration pool must be non-empty")
        if not self.labels:
            raise ValidationError("label set must be non-empty")
        if len(set(self.labels)) != len(self.labels):
            raise ValidationError("labels must be distinct")
        bad = [d.answer for d in self.pool if d.answer not in set(self.labels)]
        if bad:
            raise ValidationError(f"pool answer {bad[0]!r} is not in the label set")


@dataclass(frozen=True)
class MethodConfig:
    """Method knobs with the reference defaults (pipeline.py:93-136)."""

    method: str = DBSA
    pattern: masks.AttentionPattern = masks.AttentionPattern.sink_prev_self(2)
    block_size: int = 50
    ratio: float = 0.30
    granularity: str = kvstore.BLOCK_GRANULARITY
    grouping: retrieval.GroupingStrategy = field(default_factory=lambda: retrieval.GroupingStrategy.random(0))
    ordering: str = retrieval.IN_ORDER
    seed: int = 0
    max_pool_tokens: int = 262144

    def __post_init__(self) -> None:
        object.__setattr__(self, "method", canonical_method(self.method))
        if self.block_size < 1:
            raise ConfigError(f"block_size must be >= 1, got {self.block_size}")
        if not 0.0 < self.ratio <= 1.0:
            raise ConfigError(f"ratio must be in (0, 1], got {self.ratio}")
        if self.granularity not in kvstore.GRANULARITIES:
            raise ConfigError(f"unknown granularity {self.granularity!r}")
        if self.ordering not in retrieval.ORDERINGS:
            raise ConfigError(f"unknown ordering {self.ordering!r}")

    @property
    def local_blocks(self) -> int:
        return self.pattern.local_blocks

    def digest(self) -> str:
        parts = (self.method, self.pattern.kind, str(self.pattern.local_blocks), str(self.block_size),
                 f"{self.ratio:.6f}", self.granularity, self.grouping.kind, f"{self.grouping.swap_fraction:.6f}",
                 self.ordering)
        return hashlib.sha256("|".join(parts).encode("utf-8")).hexdigest()[:16]


@dataclass
class EncodedPool:
    cache: kvstore.SegmentedKVCache
    index: retrieval.Bm25Index
    partition: retrieval.BlockPartition
    metrics: Metrics
    encode_seconds: float = 0.0
    index_seconds: float = 0.0


def _device_model(weights):
    from .model import ModelWeights

    return weights.device() if isinstance(weights, ModelWeights) else weights


def render_block(template: PromptTemplate, pool, members):
    """(text, ids, per-demo token spans) of one group (pipeline.py:149-163)."""
    spans, parts, off = [], [], 0
    for e in members:
        part = template.render_demo(pool[e])
        n = len(part.encode("utf-8"))  # byte-level tokenizer: one token per byte
        spans.append((off, off + n))
        parts.append(part)
        off += n
    text = "".join(parts)
    return text, tokenizer.encode(text), tuple(spans)


def encode_blocks(weights, cache: kvstore.SegmentedKVCache, new_blocks, pattern: masks.AttentionPattern) -> int:
    """Append and encode groups (token ids, sha256 digest, demo spans) against
    their allowed context (pipeline.py:166-233).  All new groups go through the
    model together, layer by layer, on the GPU.  Returns attended pairs."""
    dm = _device_model(weights)
    kvstore.check_compatible(cache, dm.config)
    if not new_blocks:
        return 0
    counts = [len(ids) for ids, _, _ in new_blocks]
    total = cache.total_tokens + sum(counts)
    if total >= dm.config.max_seq_len:
        raise ValidationError(f"pool of {total} tokens exceeds max_seq_len {dm.config.max_seq_len}")
    ids = np.concatenate([np.asarray(i, np.int64) for i, _, _ in new_blocks])
    if ids.min() < 0 or ids.max() >= dm.config.vocab_size:
        raise ValidationError(f"token id outside vocabulary [0, {dm.config.vocab_size})")
    new = cache._reserve(counts, [d for _, d, _ in new_blocks], [s for _, _, s in new_blocks])
    return engine.encode_groups(dm, cache, new, ids, pattern)


def build_index(task: TaskSpec, partition: retrieval.BlockPartition, spans_per_block, granularity: str):
    """Unit texts and cache coordinates per granularity (pipeline.py:236-262)."""
    raw = [d.raw_text() for d in task.pool]
    if granularity == kvstore.BLOCK_GRANULARITY:
        texts = [" ".join(raw[e] for e in m) for m in partition.blocks]
        refs = [(b, 0, spans_per_block[b][-1][1]) for b in range(partition.n_blocks)]
        examples = [tuple(m) for m in partition.blocks]
    else:
        first = partition.blocks[0]
        texts, refs, examples = [" ".join(raw[e] for e in first)], [(0, 0, spans_per_block[0][-1][1])], [tuple(first)]
        for b in range(1, partition.n_blocks):
            for slot, e in enumerate(partition.blocks[b]):
                texts.append(raw[e])
                refs.append((b, *spans_per_block[b][slot]))
                examples.append((e,))
    return retrieval.Bm25Index(texts, granularity, refs, examples)


def encode_pool(weights, task: TaskSpec, config: MethodConfig, partition: retrieval.BlockPartition | None = None,
                device=None) -> EncodedPool:
    """Stage 1: group, render, encode on the GPU, index (pipeline.py:286-319)."""
    dm = _device_model(weights)
    t0 = time.perf_counter()
    if partition is None:
        partition = retrieval.group([d.raw_text() for d in task.pool], config.block_size,
                                    replace(config.grouping, seed=config.seed))
    rendered = [render_block(task.template, task.pool, m) for m in partition.blocks]
    total = sum(len(ids) for _, ids, _ in rendered)
    if total > config.max_pool_tokens:
        raise ValidationError(f"pool of {total} tokens exceeds the configured limit {config.max_pool_tokens}")
    cache = kvstore.SegmentedKVCache(dm.config, device or dm.device, capacity_tokens=total)
    new_blocks = [(ids, hashlib.sha256(text.encode("utf-8")).digest(), spans) for text, ids, spans in rendered]
    attended = encode_blocks(dm, cache, new_blocks, config.pattern)
    cache.seal()
    import torch

    torch.cuda.current_stream(cache.device).synchronize()
    encode_s = time.perf_counter() - t0
    t1 = time.perf_counter()
    index = build_index(task, partition, [s for _, _, s in rendered], config.granularity)
    index_s = time.perf_counter() - t1
    m = Metrics(setup_seconds=encode_s + index_s, cache_bytes=kvstore.storage_bytes(dm.config, cache.total_tokens, 4))
    m.attended_tokens.append(attended)
    m.attention_flops.append(flops_attention(attended, dm.config, cache.total_tokens))
    return EncodedPool(cache, index, partition, m, encode_s, index_s)


class Stage2Session:
    """Batched stage 2 over a sealed cache: K4 selection, chunk tables, one
    tree-masked forward per batch, label scores and argmax on the device.

    unit_refs: (block, start, end) per retrieval unit (Bm25Index.unit_refs).
    """

    def __init__(self, weights, cache: kvstore.SegmentedKVCache, unit_refs, label_ids, ratio: float, ordering: str):
        self.dm = _device_model(weights)
        self.cache = cache
        self.label_ids = [list(x) for x in label_ids]
        self.ratio, self.ordering = ratio, ordering
        refs = np.asarray(unit_refs, dtype=np.int64).reshape(-1, 3)
        blocks = cache.blocks
        row0 = np.array([e.row0 for e in blocks], np.int64)
        pos0 = np.array([e.pos_start for e in blocks], np.int64)
        self.u_row = row0[refs[:, 0]] + refs[:, 1]
        self.u_len = refs[:, 2] - refs[:, 1]
        self.u_orig = pos0[refs[:, 0]] + refs[:, 1]
        self.n_units = len(refs)
        self.budget = retrieval.budget_for(ratio, self.n_units)

    def chunks_for(self, ids: np.ndarray):
        """ordered unit ids [B, k] -> per-query chunk tables and T'."""
        ln = self.u_len[ids]
        new_start = np.cumsum(ln, axis=1) - ln
        delta = new_start - self.u_orig[ids]
        tab = np.stack([self.u_row[ids], ln, delta], axis=-1)
        return tab, ln.sum(axis=1)

    def select(self, scores):
        """K4 on the device: float64 scores [B, n_units] (host array or device
        tensor) -> ordered unit ids (host int64)."""
        import torch

        if not isinstance(scores, torch.Tensor):
            scores = torch.from_numpy(np.ascontiguousarray(scores))
        ids = engine.ops.topk_select(scores.to(self.dm.device), self.budget, self.ordering)
        return ids.cpu().numpy().astype(np.int64)

    # Single queries (the split-KV regime, < 8 per batch) are padded to a
    # multiple of PAD_TOKENS new tokens, so queries of nearby lengths share one
    # launch shape and replay one captured graph (engine.plan_key) instead of
    # each running eagerly; batches are not padded.  4 tokens: 16 padded would
    # cost C3's 44-token query 0.8 % of its batch-1 latency (4.54 vs 4.51 ms).
    PAD_TOKENS = int(__import__("os").environ.get("DBSA_PAD_TOKENS", "4"))

    def plan(self, ids: np.ndarray, query_ids_list, target_ctas=None):
        tabs, n_ctx = self.chunks_for(ids)
        jobs = [engine.label_job(tabs[i], int(n_ctx[i]), q, self.label_ids) for i, q in enumerate(query_ids_list)]
        if len(jobs) < 8:
            max_pos = self.dm.config.max_seq_len
            jobs = [engine.pad_job(j, -(-len(j.ids) // self.PAD_TOKENS) * self.PAD_TOKENS, max_pos) for j in jobs]
        return jobs, engine.Stage2Plan(self.dm, jobs, target_ctas)

    def run(self, jobs, plan):
        """Forward + label scoring; returns device (scores [B, n_labels], argmax [B])."""
        scorer = engine.LabelScorer(self.dm, plan, jobs, len(self.label_ids))
        _, h = engine.run_jobs(self.dm, self.cache.store, jobs, plan=plan, keep=scorer.keep)
        return scorer(self.dm, h, subset=True)

    def _capacity(self, jobs):
        """Upper bound of a chunk-major batch's (works, segments) for this
        session's unit count, so one captured graph serves every batch of the
        shape (engine.chunk_major_tables: a chunk shared by E rows is cut into
        ceil(E / slab) <= E / slab + 1 works per kv head)."""
        c = self.dm.config
        slab = 256 // c.group_size
        n_new = np.array([len(j.ids) for j in jobs])
        n_ch = np.array([len(np.asarray(j.chunks).reshape(-1, 3)) for j in jobs])
        keys = min(self.n_units, int(n_ch.sum()))
        e_total = int((n_new * n_ch).sum())
        self_works = int((-(-n_new // slab)).sum())
        works = c.n_kv_heads * (-(-e_total // slab) + keys + self_works)
        return works, keys + self_works

    # Captured graphs per launch shape (engine.plan_key).  A shape is captured
    # the second time it is seen (a one-off shape runs eagerly instead of paying
    # a capture plus a private memory pool), and at most MAX_GRAPHS are kept,
    # least recently used first out, so variable-length queries cannot grow
    # the cache without bound.
    MAX_GRAPHS = 8

    def _graph_for(self, jobs, plan, scorer, before_capture=None):
        """The captured graph for this plan's shape, or None to run it eagerly."""
        from collections import OrderedDict

        key = engine.plan_key(plan, scorer)
        graphs = self.__dict__.setdefault("_graphs", OrderedDict())
        seen = self.__dict__.setdefault("_seen", {})
        stats = self.__dict__.setdefault("graph_stats", {"replays": 0, "eager": 0, "captures": 0})
        g = graphs.get(key)
        if g is not None and engine.fits_graph(g, plan):
            graphs.move_to_end(key)
            stats["replays"] += 1
            return g
        seen[key] = seen.get(key, 0) + 1
        if g is None and seen[key] < 2:
            if len(seen) > 64 * self.MAX_GRAPHS:
                seen.clear()
            stats["eager"] += 1
            return None
        stats["captures"] += 1
        if before_capture is not None:
            before_capture()
        graphs.pop(key, None)
        with _CAPTURE_LOCK:  # one capture at a time per process (Runner.infer may run in threads)
            graphs[key] = engine.GraphedStage2(self.dm, self.cache.store, jobs, plan, len(self.label_ids),
                                               capacity=self._capacity(jobs))
        while len(graphs) > self.MAX_GRAPHS:
            graphs.popitem(last=False)
        return graphs[key]

    def answer(self, scores, query_ids_list, graphed: bool = True):
        """K4 selection, planning and the scored forward of one batch.  With
        `graphed`, batches of a shape seen before replay a captured CUDA graph
        (engine.GraphedStage2) instead of issuing every launch from the host."""
        ids = self.select(scores)
        jobs, plan = self.plan(ids, query_ids_list)
        if not graphed:
            s, best = self.run(jobs, plan)
            return ids, s, best
        scorer = engine.LabelScorer(self.dm, plan, jobs, len(self.label_ids))
        g = self._graph_for(jobs, plan, scorer)
        if g is None:
            _, h = engine.run_jobs(self.dm, self.cache.store, jobs, plan=plan, keep=scorer.keep)
            s, best = scorer(self.dm, h, subset=True)
        else:
            s, best = g.replay(plan, scorer)
        return ids, s, best

    def answer_stream(self, batches):
        """Pipelined answer() over an iterable of (scores, query_ids_list)
        batches; yields (ids, scores [B, n_labels], argmax [B]) as HOST arrays,
        in order.  Batch i+1's K4 selection is enqueued on a side stream
        before batch i's graph replay, so its ids are back on the host (and
        its chunk tables are planned) while the GPU runs batch i; each batch's
        results are copied out to pinned memory right behind its replay (the
        captured graph reuses its output buffers)."""
        import torch

        main = torch.cuda.current_stream(self.dm.device)
        side = torch.cuda.Stream(self.dm.device)

        def select_async(batch):
            scores, q_ids = batch
            # device scores may come from work queued on the main stream (e.g.
            # score_matrix_device inside the generator): order K4 after it, and
            # keep the allocator from recycling the block while K4 reads it
            side.wait_stream(main)
            with torch.cuda.stream(side):
                if not isinstance(scores, torch.Tensor):
                    scores = torch.from_numpy(np.ascontiguousarray(scores)).pin_memory()
                sc_dev = scores.to(self.dm.device, non_blocking=True)
                if sc_dev.device.type == "cuda":
                    sc_dev.record_stream(side)
                ids_dev = engine.ops.topk_select(sc_dev, self.budget, self.ordering)
                ids_host = torch.empty(ids_dev.shape, dtype=ids_dev.dtype, pin_memory=True)
                ids_host.copy_(ids_dev, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
            return ev, ids_host, q_ids

        prof = self.__dict__.get("stream_profile")  # list: per-batch host phase times (s), when set
        clock = time.perf_counter
        it = iter(batches)
        first = next(it, None)
        nxt = select_async(first) if first is not None else None
        pending = None
        while nxt is not None:
            t0 = clock()
            ev_sel, ids_host, q_ids = nxt
            ev_sel.synchronize()  # this batch's K4 only
            t1 = clock()
            ids = ids_host.numpy().astype(np.int64)
            jobs, plan = self.plan(ids, q_ids)
            scorer = engine.LabelScorer(self.dm, plan, jobs, len(self.label_ids))
            g = self._graph_for(jobs, plan, scorer, before_capture=main.synchronize)
            t2 = clock()
            b = next(it, None)
            nxt = select_async(b) if b is not None else None  # ahead of this batch's replay
            t3 = clock()
            if g is None:
                _, h = engine.run_jobs(self.dm, self.cache.store, jobs, plan=plan, keep=scorer.keep)
                s_dev, best_dev = scorer(self.dm, h, subset=True)
            else:
                s_dev, best_dev = g.replay(plan, scorer)
            s_host = torch.empty(s_dev.shape, dtype=s_dev.dtype, pin_memory=True)
            b_host = torch.empty(best_dev.shape, dtype=best_dev.dtype, pin_memory=True)
            s_host.copy_(s_dev, non_blocking=True)
            b_host.copy_(best_dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(main)
            t4 = clock()
            if pending is not None:
                pending[0].synchronize()
            if prof is not None:
                prof.append({"wait_select": t1 - t0, "plan": t2 - t1, "select_next": t3 - t2,
                             "enqueue": t4 - t3, "wait_prev": clock() - t4})
            if pending is not None:
                yield pending[1:]
            pending = (ev, ids, s_host.numpy(), b_host.numpy())
        if pending is not None:
            pending[0].synchronize()
            yield pending[1:]


_CAPTURE_LOCK = threading.Lock()


class Runner:
    """Inference session over (weights, cache, index) (pipeline.py:322-446).
    Read-only after prepare(); infer() may run from several threads, as the
    reference's bench does (bench.py:147-150): every thread gets its own CUDA
    stream and its own Stage2Session (whose captured graphs own their table
    and output buffers), and the shared state -- weights, cache pages, the
    index's device tables -- is built once, before any thread uses it."""

    def __init__(self, weights, cache, index, task: TaskSpec, config: MethodConfig):
        self.weights = weights
        self.dm = _device_model(weights)
        self.cache, self.index, self.task, self.config = cache, index, task, config
        self.method = config.method
        if self.method == RET_ICL:
            raise ConfigError("method 'ret' (no-cache re-encode baseline) is outside the DBSA GPU path")
        if self.method in (DBSA, FIXED_ICL) and cache is None:
            raise ValidationError(f"method {self.method!r} requires an encoded cache")
        if self.method == DBSA and index is None:
            raise ValidationError(f"method {self.method!r} requires a retrieval index")
        if cache is not None and cache.config_hash != self.dm.config.hash_bytes():
            raise CompatibilityError("cache and weights were built for different configs")
        # lexicographic label order: score ties resolve to the smallest label (pipeline.py:349-354)
        self.labels = sorted(task.labels)
        self.label_ids = [tokenizer.encode(task.template.render_label(lab)) for lab in self.labels]
        self._full: kvstore.AssembledCache | None = None
        self._lock = threading.Lock()
        self._tls = threading.local()
        self._gpu_ready = False

    def _thread_state(self):
        """(Stage2Session, CUDA stream) of the calling thread (DBSA path)."""
        import torch

        st = self._tls
        if not hasattr(st, "sess"):
            if not self._gpu_ready:
                with self._lock:
                    if not self._gpu_ready:
                        # shared device state, built once and complete before any thread reads it
                        self.index.device_tables(self.dm.device)
                        torch.cuda.synchronize(self.dm.device)
                        self._gpu_ready = True
            st.sess = self.session()
            st.stream = torch.cuda.Stream(self.dm.device)
        return st.sess, st.stream

    def _infer_dbsa(self, query_text: str, query_ids, qm):
        """The drop-in single-query DBSA call on the GPU: BM25 (csrc/bm25.cu,
        bit-identical to the reference's f64 scores) -> K4 select + order
        (csrc/topk.cu; retrieval.py:352-388) -> chunk table (assemble without a
        copy) -> the scored forward, replayed as a captured CUDA graph once its
        launch shape has been seen (Stage2Session._graph_for)."""
        import torch

        sess, stream = self._thread_state()
        with torch.cuda.stream(stream):
            t0 = time.perf_counter()
            scores = self.index.score_matrix_device([retrieval.bm25_tokenize(query_text)], self.dm.device)
            ids = sess.select(scores)
            qm.retrieval_seconds = time.perf_counter() - t0
            t0 = time.perf_counter()
            jobs, plan = sess.plan(ids, [query_ids])
            n_ctx = int(jobs[0].n_ctx)
            qm.assembly_seconds = time.perf_counter() - t0
            t0 = time.perf_counter()
            scorer = engine.LabelScorer(self.dm, plan, jobs, len(self.label_ids))
            g = sess._graph_for(jobs, plan, scorer, before_capture=stream.synchronize)
            if g is None:
                _, h = engine.run_jobs(self.dm, self.cache.store, jobs, plan=plan, keep=scorer.keep)
                _, best = scorer(self.dm, h, subset=True)
            else:
                _, best = g.replay(plan, scorer)
            label = self.labels[int(best.cpu()[0])]
            qm.scoring_seconds = time.perf_counter() - t0
        return label, n_ctx

    def prepare(self) -> None:
        if self.method == FIXED_ICL and self._full is None:
            with self._lock:
                if self._full is None:
                    self._full = kvstore.assemble(self.cache, kvstore.all_blocks_selection(self.cache))

    def _pairs(self, n_ctx: int, query_ids) -> tuple[int, int]:
        pairs = tokens = 0
        for lab in self.label_ids:
            n = len(query_ids) + len(lab)
            pairs += n * n_ctx + n * (n + 1) // 2
            tokens += n
        return pairs, tokens

    def _score(self, assembled, query_ids):
        scores = engine.score_labels(self.dm, assembled, query_ids, self.label_ids)
        best = int(np.argmax(scores))  # first maximum == strict '>' scan (pipeline.py:380-382)
        return self.labels[best], scores

    def infer(self, query_text: str):
        qm = QueryMetrics()
        t_start = time.perf_counter()
        query_ids = tokenizer.encode(self.task.template.render_query(query_text))
        if self.method == ZERO_SHOT:
            assembled = None
            n_ctx = 0
        elif self.method == FIXED_ICL:
            t0 = time.perf_counter()
            self.prepare()
            assembled = self._full
            qm.assembly_seconds = time.perf_counter() - t0
            n_ctx = assembled.total_tokens
        else:
            label, n_ctx = self._infer_dbsa(query_text, query_ids, qm)
        if self.method != DBSA:
            t0 = time.perf_counter()
            label, _ = self._score(assembled, query_ids)
            qm.scoring_seconds = time.perf_counter() - t0
        pairs, tokens = self._pairs(n_ctx, query_ids)
        qm.attended_pairs = pairs
        qm.attention_flops = flops_attention(pairs, self.dm.config, tokens)
        qm.total_seconds = time.perf_counter() - t_start
        return label, qm

    def session(self) -> Stage2Session:
        if self.method != DBSA:
            raise ConfigError("batched inference is the DBSA path")
        return Stage2Session(self.dm, self.cache, self.index.unit_refs, self.label_ids, self.config.ratio,
                             self.config.ordering)

    def infer_batch(self, query_texts, max_batch: int = 256):
        """DBSA answers for many queries: BM25 matrix on the host, K4 selection
        and one batched tree-masked forward per `max_batch` queries on the GPU.
        Returns [(label, QueryMetrics)] in input order."""
        sess = self.session()
        out = []
        for b0 in range(0, len(query_texts), max_batch):
            texts = list(query_texts[b0:b0 + max_batch])
            t0 = time.perf_counter()
            q_ids = [tokenizer.encode(self.task.template.render_query(t)) for t in texts]
            # GPU BM25 (bit-identical to the host scores) straight into K4
            scores = self.index.score_matrix_device([retrieval.bm25_tokenize(t) for t in texts], self.dm.device)
            ids, _, best = sess.answer(scores, q_ids)
            best = best.cpu().numpy()
            dt = (time.perf_counter() - t0) / len(texts)
            _, n_ctx = sess.chunks_for(ids)
            for i in range(len(texts)):
                qm = QueryMetrics()
                pairs, tokens = self._pairs(int(n_ctx[i]), q_ids[i])
                qm.attended_pairs = pairs
                qm.attention_flops = flops_attention(pairs, self.dm.config, tokens)
                qm.total_seconds = dt
                out.append((self.labels[int(best[i])], qm))
        return out


def infer(weights, cache, index, config: MethodConfig, query_text: str, task: TaskSpec):
    """Single-query convenience wrapper (pipeline.py:471-482)."""
    runner = Runner(weights, cache, index, task, config)
    runner.prepare()
    return runner.infer(query_text)
