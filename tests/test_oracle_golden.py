"""Pins the CPU oracle (oracle/dbsa_oracle.py) to golden vectors produced by
running the unmodified reference (tests/golden/make_golden.py) -- the oracle
is only trusted as a checker because these pass.  CPU only.
"""

import math

import numpy as np
import pytest

from golden_util import CASES, load, oracle_pool
from oracle import dbsa_oracle as O


@pytest.mark.parametrize("name", CASES)
def test_weights_checksum_matches_reference(name):
    meta, _ = load(name)
    w = O.init_random(O.Cfg(**meta["spec"]["model"]), meta["spec"]["weight_seed"])
    assert O.weights_checksum(w) == meta["weights_checksum"]


@pytest.mark.parametrize("name", CASES)
def test_stage1_structure_bit_exact(name):
    meta, a = load(name)
    st = oracle_pool(name)
    members = [e for b in st["partition"] for e in b]
    np.testing.assert_array_equal(members, a["partition_members"])
    np.testing.assert_array_equal([len(b) for b in st["partition"]], a["partition_sizes"])
    np.testing.assert_array_equal(st["counts"], a["block_counts"])
    allowed = O.block_mask(len(st["counts"]), "sink-prev-self", st["method"]["local_blocks"])
    np.testing.assert_array_equal(allowed.astype(np.uint8), a["block_mask"])
    assert st["attended"] == meta["attended_pairs"]
    assert O.allowed_token_pairs(allowed, st["counts"]) == meta["attended_pairs"]
    assert [list(r) for r in st["refs"]] == meta["unit_refs"]


@pytest.mark.parametrize("name", CASES)
def test_stage1_kv_samples(name):
    meta, a = load(name)
    st = oracle_pool(name)
    for layer in range(st["cfg"].n_layers):
        for b in meta["sample_blocks"]:
            k, v = st["kv"][layer][b]
            assert np.abs(k[:3] - a[f"k_l{layer}_b{b}"]).max() <= 1e-5
            assert np.abs(v[:3] - a[f"v_l{layer}_b{b}"]).max() <= 1e-5


@pytest.mark.parametrize("name", CASES)
def test_stage2_selection_scores_and_labels(name):
    meta, a = load(name)
    st = oracle_pool(name)
    c, w, m = st["cfg"], st["weights"], st["method"]
    n_check = len(meta["queries"]) if name != "c1" else 8
    for qi, q in enumerate(meta["queries"][:n_check]):
        terms = O.bm25_terms(q["query"])
        scores = [st["index"].score(terms, u) for u in range(st["index"].n)]
        np.testing.assert_array_equal(np.array(scores), a[f"q{qi}_bm25"])  # bit-exact f64
        label, lab_scores, units, n_ctx = O.infer(c, w, st["kv"], st["index"], st["refs"], st["labels"],
                                                  q["query"], m["ratio"], m["ordering"])
        np.testing.assert_array_equal(units, a[f"q{qi}_units"])
        assert n_ctx == q["assembled_tokens"]
        assert np.abs(np.array(lab_scores) - a[f"q{qi}_label_scores"]).max() <= 1e-6
        assert label == q["predicted"]


@pytest.mark.parametrize("name", CASES)
def test_forward_query_logits(name):
    """forward_query logits of the first 8 queries (model.py:400-411)."""
    meta, a = load(name)
    st = oracle_pool(name)
    for qi, q in enumerate(meta["queries"][:8]):
        units = list(a[f"q{qi}_units"])
        asm, n_ctx = O.assemble(st["cfg"], st["kv"], [st["refs"][u] for u in units])
        got = O.forward_query(st["cfg"], st["weights"], asm, n_ctx, O.encode(O.QUERY_FMT.format(query=q["query"])))
        assert np.abs(got - a[f"q{qi}_logits"]).max() <= 1e-5


def test_known_answer_vectors():
    # masks closed form 1+2+3+4(B-3) (test_masks.py:40-56) and B=60 -> 234
    for b in range(3, 201):
        assert int(O.block_mask(b, "sink-prev-self", 2).sum()) == 1 + 2 + 3 + 4 * (b - 3)
    assert int(O.block_mask(60, "sink-prev-self", 2).sum()) == 234
    # context ids (test_masks.py:81-85)
    assert O.context_ids(O.block_mask(8, "sink-prev-self", 2), 5) == (0, 3, 4)
    assert O.context_ids(O.block_mask(8, "sink-prev-self", 2), 0) == ()
    # sparsity at B=69, 30 tok/block in [0.88, 0.92] (test_masks.py:99-102)
    allowed = O.block_mask(69, "sink-prev-self", 2)
    total = 69 * 30
    sp = 1 - O.allowed_token_pairs(allowed, [30] * 69) / (total * (total + 1) // 2)
    assert 0.88 <= sp <= 0.92
    # select budget = ceil(ratio * n), anchor first (retrieval.py:367-370)
    for n in (1, 7, 20, 60):
        for r in (0.1, 0.3, 0.5, 1.0):
            sel = O.select([0.0] * n, r)
            assert sel[0] == 0 and len(sel) == math.ceil(r * n)
