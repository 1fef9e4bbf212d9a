"""Generate the golden parity fixtures by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the reference package read-only from /root/reference/pkg/src and
writes tests/golden/<name>.npz + <name>.json.  The GPU box never runs this
(the reference is not there); tests read the committed fixtures.

Each fixture records, for one (model config, task, method config):
  weights checksum (model.ModelWeights.checksum, model.py:151-156), the block
  partition, per-block token counts, block mask (masks.py:80-99), attended
  pairs (pipeline.py:231-232), K/V samples of the cache (kvstore.py:59-60),
  and per test query: BM25 scores (retrieval.py:129-141), ordered unit ids
  (retrieval.py:352-388), assembled length, per-label scores
  (model.score_label, model.py:420-443) and the predicted label
  (pipeline.py:369-384); plus forward_query logits of the first 8 queries
  (model.py:400-411).
"""

from __future__ import annotations

import json
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

CASES = {
    # C1 of BASELINE.json: the CLI init-model defaults (cli.py:282-288), 256 demos, groups of 16.
    "c1": dict(model=dict(d_model=64, n_layers=2, n_heads=4, n_kv_heads=2, head_dim=16, ffn_dim=128),
               weight_seed=0, task=dict(n_demos=256, n_tests=32, n_labels=4, seed=0),
               method=dict(block_size=16, ratio=0.3, seed=0)),
    # head_dim 128 with 4 query heads per kv head (the Llama-3.1-8B GQA factor), 2 M-tiles per work.
    "g128": dict(model=dict(d_model=512, n_layers=2, n_heads=4, n_kv_heads=1, head_dim=128, ffn_dim=512),
                 weight_seed=1, task=dict(n_demos=64, n_tests=8, n_labels=4, seed=1),
                 method=dict(block_size=8, ratio=0.3, seed=1)),
    # MHA head_dim 64, example granularity, low-to-high ordering, sink-prev-self(1).
    "m64ex": dict(model=dict(d_model=256, n_layers=2, n_heads=4, n_kv_heads=4, head_dim=64, ffn_dim=256),
                  weight_seed=2, task=dict(n_demos=48, n_tests=8, n_labels=3, seed=2),
                  method=dict(block_size=6, ratio=0.5, seed=2, granularity="example", ordering="low-to-high",
                              local_blocks=1)),
}


def run_case(name: str, spec: dict) -> None:
    from dbsa import kvstore, masks, model, pipeline, retrieval, synthetic, tokenizer

    cfg = model.ModelConfig(vocab_size=tokenizer.VOCAB_SIZE, **spec["model"])
    weights = model.init_random(cfg, seed=spec["weight_seed"])
    data = synthetic.generate_recall_task(**spec["task"])
    task = pipeline.TaskSpec(data.pool, data.labels)
    m = dict(spec["method"])
    j = m.pop("local_blocks", 2)
    mc = pipeline.MethodConfig(pattern=masks.AttentionPattern.sink_prev_self(j), **m)
    t0 = time.perf_counter()
    enc = pipeline.encode_pool(weights, task, mc)
    t_enc = time.perf_counter() - t0
    cache, index = enc.cache, enc.index
    counts = [e.token_count for e in cache.blocks]
    bm = masks.build_block_mask(cache.n_blocks, mc.pattern)

    arrays: dict[str, np.ndarray] = {
        "partition_members": np.array([e for b in enc.partition.blocks for e in b], np.int64),
        "partition_sizes": np.array([len(b) for b in enc.partition.blocks], np.int64),
        "block_counts": np.array(counts, np.int64),
        "block_mask": bm.allowed.astype(np.uint8),
    }
    sample_blocks = sorted({0, 1, cache.n_blocks - 1})
    for layer in range(cfg.n_layers):
        for b in sample_blocks:
            k, v = cache.segment(layer, b)
            arrays[f"k_l{layer}_b{b}"] = np.asarray(k[:3], np.float32)
            arrays[f"v_l{layer}_b{b}"] = np.asarray(v[:3], np.float32)

    queries = []
    t1 = time.perf_counter()
    runner = pipeline.Runner(weights, cache, index, task, mc)
    runner.prepare()
    for qi, test in enumerate(data.tests):
        label, qm = runner.infer(test.query)
        terms = retrieval.bm25_tokenize(test.query)
        scores = [index.score(terms, u) for u in range(index.n_docs)]
        sel = retrieval.order(retrieval.select(index, test.query, mc.ratio, mc.granularity), mc.ordering)
        asm = kvstore.assemble(cache, sel)
        q_ids = tokenizer.encode(task.template.render_query(test.query))
        lab_scores = [model.score_label(weights, asm, q_ids, tokenizer.encode(task.template.render_label(lab)))
                      for lab in sorted(task.labels)]
        arrays[f"q{qi}_bm25"] = np.array(scores, np.float64)
        arrays[f"q{qi}_units"] = np.array(sel.unit_ids, np.int64)
        arrays[f"q{qi}_label_scores"] = np.array(lab_scores, np.float64)
        if qi < 8:  # forward_query logits (model.py:400-411) of the first 8 queries
            seq = model.TokenSequence.at_offset(q_ids, asm.total_tokens)
            arrays[f"q{qi}_logits"] = model.forward_query(weights, asm, seq).astype(np.float32)
        queries.append(dict(query=test.query, answer=test.answer, predicted=label, assembled_tokens=asm.total_tokens,
                            attended_pairs=qm.attended_pairs))
    t_inf = time.perf_counter() - t1

    meta = dict(name=name, spec=spec, weights_checksum=weights.checksum(), config_hash=cfg.hash_bytes().hex(),
                labels=list(task.labels), n_blocks=cache.n_blocks, total_tokens=cache.total_tokens,
                attended_pairs=int(enc.metrics.attended_tokens[0]), n_units=index.n_docs,
                unit_refs=[list(r) for r in index.unit_refs], queries=queries, sample_blocks=sample_blocks,
                reference_seconds=dict(encode=t_enc, infer_total=t_inf))
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    (OUT / f"{name}.json").write_text(json.dumps(meta, indent=1))
    print(f"{name}: {cache.n_blocks} blocks, {cache.total_tokens} tokens, encode {t_enc:.2f}s, "
          f"infer {t_inf:.2f}s for {len(queries)} queries")


def make_cache_file() -> None:
    """A small DBSACACH file written by the reference's serialize
    (kvstore.py:238-258) for the cache-file parity tests."""
    from dbsa import kvstore, masks, model, pipeline, synthetic, tokenizer

    spec = CASES["c1"]
    cfg = model.ModelConfig(vocab_size=tokenizer.VOCAB_SIZE, **spec["model"])
    weights = model.init_random(cfg, seed=0)
    data = synthetic.generate_recall_task(n_demos=24, n_tests=2, n_labels=4, seed=3)
    task = pipeline.TaskSpec(data.pool, data.labels)
    mc = pipeline.MethodConfig(block_size=4, ratio=0.5, seed=3, granularity="example",
                               pattern=masks.AttentionPattern.sink_prev_self(2))
    enc = pipeline.encode_pool(weights, task, mc)
    kvstore.serialize(enc.cache, OUT / "cache_tiny.dbsacache")
    meta = dict(model=spec["model"], weight_seed=0, task=dict(n_demos=24, n_tests=2, n_labels=4, seed=3),
                method=dict(block_size=4, ratio=0.5, seed=3, granularity="example"), n_blocks=enc.cache.n_blocks,
                total_tokens=enc.cache.total_tokens,
                file_size=(OUT / "cache_tiny.dbsacache").stat().st_size)
    (OUT / "cache_tiny.json").write_text(json.dumps(meta, indent=1))
    print(f"cache_tiny: {enc.cache.n_blocks} blocks, {enc.cache.total_tokens} tokens, {meta['file_size']} bytes")


def main(names=None):
    sys.path.insert(0, str(REF))
    if names == ["cache"]:
        make_cache_file()
        return
    for name in names or CASES:
        run_case(name, CASES[name])
    make_cache_file()


if __name__ == "__main__":
    main(sys.argv[1:] or None)
