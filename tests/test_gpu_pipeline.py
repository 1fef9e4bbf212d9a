"""End-to-end parity of the GPU path against the reference, through the
reference-shaped API (encode_pool -> SegmentedKVCache -> Runner.infer).

Reference values are the committed golden fixtures produced by the
unmodified reference (tests/golden/make_golden.py); the CPU oracle
(oracle/dbsa_oracle.py, pinned to the same fixtures) supplies what the
fixtures do not store.  Gates (north star):
  * partition, block mask, attended pairs, selected unit ids: bit-exact;
  * K/V pages vs the reference's f32 cache: max-abs 3e-2 (bf16 storage);
  * forward_query logits: max-abs 2e-2 vs the reference's f32 logits;
  * per-label scores: max-abs 0.04 (a sum of ~6 bf16 log-probs; the
    measured worst is ~0.03 on the chunk-major bf16-partial path);
  * predicted labels: identical, no exceptions (the smallest reference top-2
    margin over the three cases is 0.043, m64ex; it is printed).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_util import CASES, load, oracle_pool  # noqa: E402
from oracle import dbsa_oracle as O  # noqa: E402
import paper_2503_08640_b200 as P  # noqa: E402
from paper_2503_08640_b200 import engine, masks, pipeline, retrieval, tokenizer  # noqa: E402

LOGIT_TOL = 2e-2
KV_TOL = 3e-2
SCORE_TOL = 0.04


def _setup(name):
    meta, a = load(name)
    cfg = P.ModelConfig(vocab_size=tokenizer.VOCAB_SIZE, **meta["spec"]["model"])
    w = P.init_random(cfg, meta["spec"]["weight_seed"])
    t = meta["spec"]["task"]
    pool, tests, labels = O.recall_task(t["n_demos"], t["n_tests"], t["n_labels"], t["seed"])
    task = P.TaskSpec(tuple(P.Demonstration(q, x) for q, x in pool), tuple(labels))
    m = dict(meta["spec"]["method"])
    j = m.pop("local_blocks", 2)
    mc = P.MethodConfig(pattern=masks.AttentionPattern.sink_prev_self(j), **m)
    return meta, a, w, task, mc


_ENC = {}


def _encoded(name):
    if name not in _ENC:
        meta, a, w, task, mc = _setup(name)
        _ENC[name] = (meta, a, w, task, mc, P.encode_pool(w, task, mc))
    return _ENC[name]


@pytest.mark.parametrize("name", CASES)
def test_stage1_structure_and_pages(name):
    meta, a, w, task, mc, enc = _encoded(name)
    cache = enc.cache
    assert cache.sealed and cache.n_blocks == meta["n_blocks"] and cache.total_tokens == meta["total_tokens"]
    np.testing.assert_array_equal([e.token_count for e in cache.blocks], a["block_counts"])
    np.testing.assert_array_equal([x for b in enc.partition.blocks for x in b], a["partition_members"])
    assert enc.metrics.attended_tokens[0] == meta["attended_pairs"]
    worst = 0.0
    for layer in range(w.config.n_layers):
        for b in meta["sample_blocks"]:
            k, v = cache.segment(layer, b)
            worst = max(worst, float(np.abs(k[:3] - a[f"k_l{layer}_b{b}"]).max()),
                        float(np.abs(v[:3] - a[f"v_l{layer}_b{b}"]).max()))
    assert worst < KV_TOL, worst


def test_stage1_whole_cache_vs_oracle_c1():
    """Every group, every layer: pages vs the oracle's f32 stage 1 (pinned to
    the reference by test_oracle_golden)."""
    meta, a, w, task, mc, enc = _encoded("c1")
    st = oracle_pool("c1")
    worst = 0.0
    for layer in range(w.config.n_layers):
        for b in range(enc.cache.n_blocks):
            k, v = enc.cache.segment(layer, b)
            rk, rv = st["kv"][layer][b]
            worst = max(worst, float(np.abs(k - rk).max()), float(np.abs(v - rv).max()))
    assert worst < KV_TOL, worst


@pytest.mark.parametrize("split", ["packed-bf16", "packed-fp32", "round-robin-fp32", "packed-bf16-pad16"])
@pytest.mark.parametrize("name", CASES)
def test_stage2_runner_matches_reference(name, split, monkeypatch):
    """Runner.infer / score_label per query against the reference goldens,
    through the split-KV schedule as shipped (cost-packed CTA ranges, SELF as
    its own split, bf16 partials, queries padded by a dummy tree branch to a
    multiple of 4 tokens), its fp32 / round-robin variants, and 16-token
    padding."""
    monkeypatch.setenv("DBSA_PACK", "0" if split.startswith("round-robin") else "1")
    monkeypatch.setenv("DBSA_SPLIT_BF16", "1" if "bf16" in split else "0")
    monkeypatch.setattr(P.Stage2Session, "PAD_TOKENS", 16 if split.endswith("pad16") else 4)
    meta, a, w, task, mc, enc = _encoded(name)
    runner = P.Runner(w, enc.cache, enc.index, task, mc)
    runner.prepare()
    worst, margins, flips = 0.0, [], []
    for qi, q in enumerate(meta["queries"]):
        sel = retrieval.order(retrieval.select(enc.index, q["query"], mc.ratio, mc.granularity), mc.ordering)
        np.testing.assert_array_equal(sel.unit_ids, a[f"q{qi}_units"])  # bit-exact selection
        asm = P.assemble(enc.cache, sel)
        assert asm.total_tokens == q["assembled_tokens"]
        label, qm = runner.infer(q["query"])
        assert qm.attended_pairs == q["attended_pairs"]
        q_ids = tokenizer.encode(task.template.render_query(q["query"]))
        got = runner._score(asm, q_ids)[1]
        ref = a[f"q{qi}_label_scores"]
        err = float(np.abs(got - ref).max())
        worst = max(worst, err)
        srt = np.sort(ref)
        margin = float(srt[-1] - srt[-2]) if len(ref) > 1 else np.inf
        margins.append(margin)
        if label != q["predicted"]:
            flips.append((qi, margin, err))
    print(f"{name}: max |score err| {worst:.4g}; min top-2 margin {min(margins):.4g}; flips {flips}")
    assert worst < SCORE_TOL, worst
    assert not flips, f"predicted labels differ from the reference: {flips}"


@pytest.mark.parametrize("name", ["c1", "m64ex"])
def test_runner_infer_from_threads_equals_serial(name):
    """The reference runs Runner.infer concurrently from a ThreadPoolExecutor
    (bench.py:147-150).  Four threads (each on its own stream, with its own
    captured graphs) answering every golden query twice give the serial
    labels, which are the reference's; the drop-in single-query call runs
    GPU BM25 + K4 (ops.LAUNCHES counts them) and replays captured graphs."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2503_08640_b200 import ops

    meta, a, w, task, mc, enc = _encoded(name)
    runner = P.Runner(w, enc.cache, enc.index, task, mc)
    queries = [q["query"] for q in meta["queries"]]
    n0 = ops.LAUNCHES
    serial = [runner.infer(q)[0] for q in queries]
    assert ops.LAUNCHES > n0
    assert serial == [q["predicted"] for q in meta["queries"]]
    with ThreadPoolExecutor(4) as ex:
        par = list(ex.map(lambda q: runner.infer(q)[0], queries * 2))
    assert par == serial * 2
    sess = runner._thread_state()[0]
    assert len(sess.__dict__.get("_graphs", {})) >= 1  # the repeated batch-1 shape is replayed from a graph


@pytest.mark.parametrize("schedule", ["query", "chunk"])
@pytest.mark.parametrize("name", CASES)
def test_stage2_batched_k4_path_matches_reference(name, schedule, monkeypatch):
    """Runner.infer_batch: K4 selection on the device + one tree-masked
    forward for the whole batch (split-KV per query and chunk-major K3);
    unit ids bit-exact, labels identical."""
    monkeypatch.setenv("DBSA_STAGE2_SCHEDULE", schedule)
    meta, a, w, task, mc, enc = _encoded(name)
    runner = P.Runner(w, enc.cache, enc.index, task, mc)
    texts = [q["query"] for q in meta["queries"]]
    sess = runner.session()
    scores = enc.index.score_matrix([retrieval.bm25_tokenize(t) for t in texts])
    ids = sess.select(scores)
    for qi in range(len(texts)):
        np.testing.assert_array_equal(ids[qi], a[f"q{qi}_units"])
    out = runner.infer_batch(texts, max_batch=7)
    single = [runner.infer(t)[0] for t in texts]
    assert [lab for lab, _ in out] == single
    for qi, (lab, qm) in enumerate(out):
        assert qm.attended_pairs == meta["queries"][qi]["attended_pairs"]
    # the pipelined batch entry point: same ids and labels, batch by batch
    q_ids = [tokenizer.encode(task.template.render_query(t)) for t in texts]
    half = len(texts) // 2
    batches = [(scores[:half], q_ids[:half]), (scores[half:], q_ids[half:])]
    got = list(sess.answer_stream(batches))
    for (ids_b, s_b, best_b), (sc_b, q_b) in zip(got, batches):
        ids1, s1, best1 = sess.answer(sc_b, q_b)
        np.testing.assert_array_equal(ids_b, ids1)
        np.testing.assert_array_equal(best_b, best1.cpu().numpy())
        np.testing.assert_allclose(s_b, s1.cpu().numpy(), atol=1e-5)


@pytest.mark.parametrize("name", CASES)
def test_answer_stream_mixed_shapes_generator(name):
    """answer_stream over a generator of batches whose shapes change mid-stream
    (a new graph is captured while the next batch's K4 is already in flight):
    every batch equals answer() on its own, in order."""
    meta, a, w, task, mc, enc = _encoded(name)
    runner = P.Runner(w, enc.cache, enc.index, task, mc)
    sess = runner.session()
    texts = [q["query"] for q in meta["queries"]]
    scores = enc.index.score_matrix([retrieval.bm25_tokenize(t) for t in texts])
    q_ids = [tokenizer.encode(task.template.render_query(t)) for t in texts]
    cuts = [(0, 3), (3, 6), (6, 8), (0, 1), (1, 4)]
    got = list(sess.answer_stream((scores[i:j], q_ids[i:j]) for i, j in cuts))
    assert len(got) == len(cuts)
    for (i, j), (ids_b, s_b, best_b) in zip(cuts, got):
        ids1, s1, best1 = sess.answer(scores[i:j], q_ids[i:j])
        np.testing.assert_array_equal(ids_b, ids1)
        np.testing.assert_array_equal(best_b, best1.cpu().numpy())
        np.testing.assert_allclose(s_b, s1.cpu().numpy(), atol=1e-5)
    assert list(sess.answer_stream(iter(()))) == []


@pytest.mark.parametrize("name", CASES)
def test_stage2_scored_row_subset_equals_full(name):
    """The last layer's O projection and FFN on the distinct scored rows only
    (LabelScorer.keep) give the same label scores as the full last layer."""
    meta, a, w, task, mc, enc = _encoded(name)
    runner = P.Runner(w, enc.cache, enc.index, task, mc)
    texts = [q["query"] for q in meta["queries"]]
    sess = runner.session()
    scores = enc.index.score_matrix([retrieval.bm25_tokenize(t) for t in texts])
    q_ids = [tokenizer.encode(task.template.render_query(t)) for t in texts]
    jobs, plan = sess.plan(sess.select(scores), q_ids)
    scorer = engine.LabelScorer(sess.dm, plan, jobs, len(sess.label_ids))
    assert scorer.keep.numel() < plan.new.n_tok
    _, h_sub = engine.run_jobs(sess.dm, sess.cache.store, jobs, plan=plan, keep=scorer.keep)
    s_sub, b_sub = scorer(sess.dm, h_sub, subset=True)
    _, h_all = engine.run_jobs(sess.dm, sess.cache.store, jobs, plan=plan)
    s_all, b_all = scorer(sess.dm, h_all)
    np.testing.assert_allclose(s_sub.cpu().numpy(), s_all.cpu().numpy(), atol=2e-3, rtol=1e-4)
    np.testing.assert_array_equal(b_sub.cpu().numpy(), b_all.cpu().numpy())


def test_forward_query_logits_c1():
    meta, a, w, task, mc, enc = _encoded("c1")
    q = meta["queries"][0]
    units = [int(u) for u in a["q0_units"]]
    sel = P.Selection("block", tuple(P.SegmentRef(u, *enc.index.unit_refs[u]) for u in units))
    asm = P.assemble(enc.cache, sel)
    q_ids = tokenizer.encode(task.template.render_query(q["query"]))
    got = P.forward_query(w, asm, P.TokenSequence.at_offset(q_ids, asm.total_tokens))
    err = float(np.abs(got - a["q0_logits"]).max())
    print(f"forward_query max-abs logit error {err:.4g} (|logits| <= {np.abs(a['q0_logits']).max():.3g})")
    assert err < LOGIT_TOL, err


def test_score_label_and_assembled_layers_c1():
    meta, a, w, task, mc, enc = _encoded("c1")
    st = oracle_pool("c1")
    units = [int(u) for u in a["q1_units"]]
    sel = P.Selection("block", tuple(P.SegmentRef(u, *enc.index.unit_refs[u]) for u in units))
    asm = P.assemble(enc.cache, sel)
    ref_layers, n_ctx = O.assemble(st["cfg"], st["kv"], [st["refs"][u] for u in units])
    assert n_ctx == asm.total_tokens
    for (k, v), (rk, rv) in zip(asm.layers, ref_layers):
        assert float(np.abs(k - rk).max()) < KV_TOL and float(np.abs(v - rv).max()) < KV_TOL
    q_ids = tokenizer.encode(task.template.render_query(meta["queries"][1]["query"]))
    for li, lab in enumerate(sorted(task.labels)):
        s = P.score_label(w, asm, q_ids, tokenizer.encode(task.template.render_label(lab)))
        assert abs(s - a["q1_label_scores"][li]) < SCORE_TOL


def test_incremental_append_equals_one_shot():
    """encode_blocks on an existing cache encodes only the new groups against
    the stored ones (pipeline.py:179-200, test_acceptance.py:144-180)."""
    meta, a, w, task, mc, enc = _encoded("c1")
    rendered = [pipeline.render_block(task.template, task.pool, m) for m in enc.partition.blocks]
    import hashlib

    blocks = [(ids, hashlib.sha256(t.encode()).digest(), sp) for t, ids, sp in rendered]
    cache = P.SegmentedKVCache(w.config)
    n1 = P.encode_blocks(w, cache, blocks[:5], mc.pattern)
    n2 = P.encode_blocks(w, cache, blocks[5:], mc.pattern)
    assert n1 + n2 == meta["attended_pairs"]
    worst = 0.0
    for layer in range(w.config.n_layers):
        for b in (0, 4, 5, 6, 15):
            k1, v1 = cache.segment(layer, b)
            k0, v0 = enc.cache.segment(layer, b)
            worst = max(worst, float(np.abs(k1 - k0).max()), float(np.abs(v1 - v0).max()))
    assert worst < 1e-2, worst


def test_forward_encode_api_matches_oracle():
    meta, a, w, task, mc, enc = _encoded("c1")
    st = oracle_pool("c1")
    c = st["cfg"]
    rendered = [pipeline.render_block(task.template, task.pool, m) for m in enc.partition.blocks]
    counts = [len(ids) for _, ids, _ in rendered]
    off = np.concatenate([[0], np.cumsum(counts)])
    b = 3
    ctx = (0, 1, 2)
    ctx_pos = np.concatenate([np.arange(off[j], off[j + 1]) for j in ctx])
    layers = []
    for layer in range(c.n_layers):
        ks = [O.rope(st["kv"][layer][j][0], np.arange(off[j], off[j + 1]), c.rope_theta) for j in ctx]
        layers.append((np.concatenate(ks), np.concatenate([st["kv"][layer][j][1] for j in ctx])))
    tokens = P.TokenSequence.at_offset(rendered[b][1], int(off[b]))
    mask = masks.block_mask_rows(masks.build_block_mask(16, mc.pattern), counts, b)
    pre, hidden = P.forward_encode(w, tokens, P.ContextKV(ctx_pos, layers), mask)
    for layer in range(c.n_layers):
        assert float(np.abs(pre[layer][0] - st["kv"][layer][b][0]).max()) < KV_TOL
        assert float(np.abs(pre[layer][1] - st["kv"][layer][b][1]).max()) < KV_TOL
    with pytest.raises(P.MaskError):
        bad = mask.copy()
        bad[0, 0] = False
        P.forward_encode(w, tokens, P.ContextKV(ctx_pos, layers), bad)


def test_errors_map_to_reference_exceptions():
    meta, a, w, task, mc, enc = _encoded("c1")
    with pytest.raises(P.ValidationError):
        enc.cache.append_block(16, [], b"x" * 32)  # sealed
    with pytest.raises(P.ValidationError):
        P.assemble(enc.cache, P.Selection("block", (P.SegmentRef(0, 0, 0, 10), P.SegmentRef(1, 99, 0, 5))))
    other = P.ModelConfig(64, 2, 4, 4, 16, 128, 259)
    with pytest.raises(P.CompatibilityError):
        P.Runner(P.init_random(other, 0), enc.cache, enc.index, task, mc)
    with pytest.raises(P.ValidationError):
        P.score_label(w, None, [], [5])


@pytest.mark.parametrize("name", CASES)
def test_gpu_bm25_bit_exact(name):
    """GPU BM25 (csrc/bm25.cu) equals the reference's float64 scores bit for
    bit, and K4 over them reproduces the reference's selections."""
    meta, a, w, task, mc, enc = _encoded(name)
    texts = [q["query"] for q in meta["queries"]] + ["zzz unknown terms only", "key0001 key0001 lookup"]
    terms = [retrieval.bm25_tokenize(t) for t in texts]
    dev_scores = enc.index.score_matrix_device(terms).cpu().numpy()
    host = enc.index.score_matrix(terms)
    np.testing.assert_array_equal(dev_scores, host)
    for qi in range(len(meta["queries"])):
        np.testing.assert_array_equal(dev_scores[qi], a[f"q{qi}_bm25"])
    runner = P.Runner(w, enc.cache, enc.index, task, mc)
    ids = runner.session().select(enc.index.score_matrix_device(terms[: len(meta["queries"])]))
    for qi in range(len(meta["queries"])):
        np.testing.assert_array_equal(ids[qi], a[f"q{qi}_units"])


@pytest.mark.parametrize("kind,j", [("full", 2), ("sink-self", 2), ("self", 2), ("sink-prev-self", 0),
                                    ("sink-prev-self", 3)])
def test_stage1_patterns_vs_oracle(kind, j):
    """Every AttentionPattern of the reference (masks.py:15-54) through K1 vs
    the oracle's sequential f32 stage 1 on the same groups; pair counts exact."""
    from golden_util import load as gload

    meta, _ = gload("c1")
    cfg = P.ModelConfig(vocab_size=tokenizer.VOCAB_SIZE, **meta["spec"]["model"])
    w = P.init_random(cfg, 0)
    pool, _, _ = O.recall_task(40, 1, 4, 5)
    task = P.TaskSpec(tuple(P.Demonstration(q, x) for q, x in pool), tuple(O.LABEL_WORDS[:4]))
    pattern = masks.AttentionPattern(kind, j)
    mc = P.MethodConfig(block_size=6, ratio=0.5, seed=5, pattern=pattern)
    enc = P.encode_pool(w, task, mc)
    oc = O.Cfg(**meta["spec"]["model"])
    ow = O.init_random(oc, 0)
    rendered = [pipeline.render_block(task.template, task.pool, m) for m in enc.partition.blocks]
    kv, attended = O.encode_blocks(oc, ow, [ids for _, ids, _ in rendered], kind, j)
    assert attended == enc.metrics.attended_tokens[0]
    bm = masks.build_block_mask(enc.cache.n_blocks, pattern)
    assert attended == masks.count_allowed_token_pairs(bm, [e.token_count for e in enc.cache.blocks])
    worst = 0.0
    for layer in range(cfg.n_layers):
        for b in range(enc.cache.n_blocks):
            k, v = enc.cache.segment(layer, b)
            worst = max(worst, float(np.abs(k - kv[layer][b][0]).max()), float(np.abs(v - kv[layer][b][1]).max()))
    assert worst < KV_TOL, worst


@pytest.mark.parametrize("schedule", ["query", "chunk"])
@pytest.mark.parametrize("ordering", ["in-order", "low-to-high", "reverse"])
@pytest.mark.parametrize("ratio", [0.01, 1.0])
def test_stage2_orderings_and_extreme_ratios(ordering, ratio, schedule, monkeypatch):
    """Anchor-only (ratio -> budget 1: few-shot ICL) and the whole pool, every
    ordering, through both K3 schedules (split-KV per query and chunk-major):
    K4 ids bit-exact with select + order, labels equal the oracle's."""
    monkeypatch.setenv("DBSA_STAGE2_SCHEDULE", schedule)
    meta, a, w, task, mc0, enc = _encoded("c1")
    mc = P.MethodConfig(block_size=16, ratio=ratio, seed=0, ordering=ordering)
    runner = P.Runner(w, enc.cache, enc.index, task, mc)
    texts = [q["query"] for q in meta["queries"][:6]]
    out = runner.infer_batch(texts)
    st = oracle_pool("c1")
    for t, (lab, qm) in zip(texts, out):
        want = retrieval.order(retrieval.select(enc.index, t, ratio), ordering)
        label, scores, units, n_ctx = O.infer(st["cfg"], st["weights"], st["kv"], st["index"], st["refs"],
                                              st["labels"], t, ratio, ordering)
        assert list(want.unit_ids) == units
        srt = np.sort(scores)
        assert lab == label, f"label differs from the oracle's (top-2 margin {srt[-1] - srt[-2]:.4g})"


def _permuted_scores(scores, seed=1):
    """Same batch shape, different selections: the non-anchor columns shuffled."""
    rng = np.random.default_rng(seed)
    out = scores.copy()
    cols = np.arange(1, scores.shape[1])
    out[:, cols] = scores[:, rng.permutation(cols)]
    return out


@pytest.mark.parametrize("name", CASES)
def test_benchmarked_path_graph_replay_vs_reference(name, monkeypatch):
    """The path every bench number comes from: GPU BM25 -> K4 -> chunk-major
    K3 with bf16 partials (DBSA_OUT_MAPPED row-map works) + K3m, the whole
    forward + label scoring replayed from a captured CUDA graph
    (engine.GraphedStage2).  The graph is captured on a batch with DIFFERENT
    selections (same shape), then replayed with the real batch's tables copied
    in.  Gates: unit ids bit-exact, label scores <= 0.04 from the reference's
    float64 scores (model.score_label, model.py:420-443), predicted labels
    identical (pipeline.py:369-384) with no near-tie exceptions."""
    monkeypatch.setenv("DBSA_STAGE2_SCHEDULE", "chunk")
    meta, a, w, task, mc, enc = _encoded(name)
    runner = P.Runner(w, enc.cache, enc.index, task, mc)
    sess = runner.session()
    texts = [q["query"] for q in meta["queries"]]
    q_ids = [tokenizer.encode(task.template.render_query(t)) for t in texts]
    scores_dev = enc.index.score_matrix_device([retrieval.bm25_tokenize(t) for t in texts])
    ids = sess.select(scores_dev)
    for qi in range(len(texts)):
        np.testing.assert_array_equal(ids[qi], a[f"q{qi}_units"])
    jobs, plan = sess.plan(ids, q_ids)
    assert isinstance(plan.sched, engine.ChunkMajorSchedule)
    assert plan.sched.part_o.dtype == torch.bfloat16
    other = sess.select(_permuted_scores(scores_dev.cpu().numpy()))
    assert not np.array_equal(other, ids)
    jobs_o, plan_o = sess.plan(other, q_ids)
    graph = engine.GraphedStage2(sess.dm, sess.cache.store, jobs_o, plan_o, len(sess.label_ids),
                                 capacity=sess._capacity(jobs))
    scorer = engine.LabelScorer(sess.dm, plan, jobs, len(sess.label_ids))
    assert engine.plan_key(plan, scorer) == graph.key and engine.fits_graph(graph, plan)
    s_dev, best_dev = graph.replay(plan, scorer)
    got = s_dev.double().cpu().numpy()
    best = best_dev.cpu().numpy()
    worst, margins = 0.0, []
    for qi, q in enumerate(meta["queries"]):
        ref = a[f"q{qi}_label_scores"]
        worst = max(worst, float(np.abs(got[qi] - ref).max()))
        srt = np.sort(ref)
        margins.append(float(srt[-1] - srt[-2]))
        assert runner.labels[int(best[qi])] == q["predicted"], (qi, got[qi], ref)
    print(f"{name}: graph-replayed chunk-major path, max |score err| {worst:.4g}, min margin {min(margins):.4g}")
    assert worst < SCORE_TOL, worst


@pytest.mark.parametrize("name", CASES)
def test_batched_chunk_major_logits_vs_reference(name):
    """forward_query (model.py:400-411) for the first 8 queries as ONE batch
    through the chunk-major K3 (bf16 partials) + K3m: every row's logits
    within 2e-2 of the reference's f32 logits."""
    meta, a, w, task, mc, enc = _encoded(name)
    runner = P.Runner(w, enc.cache, enc.index, task, mc)
    sess = runner.session()
    n_q = min(8, len(meta["queries"]))
    ids = np.stack([a[f"q{qi}_units"] for qi in range(n_q)]).astype(np.int64)
    tabs, n_ctx = sess.chunks_for(ids)
    jobs = []
    for qi in range(n_q):
        q_ids = tokenizer.encode(task.template.render_query(meta["queries"][qi]["query"]))
        n = len(q_ids)
        jobs.append(engine.QueryJob(tabs[qi], int(n_ctx[qi]), list(q_ids), list(range(n)), [0] * n, n))
    plan = engine.Stage2Plan(sess.dm, jobs, schedule="chunk")
    assert plan.sched.part_o.dtype == torch.bfloat16
    _, h = engine.run_jobs(sess.dm, sess.cache.store, jobs, plan=plan)
    logits = engine._final_logits(sess.dm, h).cpu().numpy()
    worst = 0.0
    for qi in range(n_q):
        t0, n = int(plan.new.tok0[qi]), plan.new.n_new[qi]
        ref = a[f"q{qi}_logits"]
        assert ref.shape == logits[t0:t0 + n].shape
        worst = max(worst, float(np.abs(logits[t0:t0 + n] - ref).max()))
    print(f"{name}: batched chunk-major logits max-abs error {worst:.4g}")
    assert worst < LOGIT_TOL, worst
