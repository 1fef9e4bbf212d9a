"""Loading helpers for the committed reference fixtures (tests/golden/*)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = ("c1", "g128", "m64ex")


@lru_cache(maxsize=None)
def load(name: str):
    meta = json.loads((GOLDEN / f"{name}.json").read_text())
    arrays = dict(np.load(GOLDEN / f"{name}.npz"))
    return meta, arrays


def oracle_cfg(meta):
    from oracle import dbsa_oracle as O

    return O.Cfg(**meta["spec"]["model"])


def method(meta):
    m = dict(meta["spec"]["method"])
    return dict(block_size=m["block_size"], ratio=m["ratio"], seed=m["seed"],
                granularity=m.get("granularity", "block"), ordering=m.get("ordering", "in-order"),
                local_blocks=m.get("local_blocks", 2))


@lru_cache(maxsize=None)
def oracle_pool(name: str):
    """Run the oracle's stage 1 for a golden case (cached per session)."""
    from oracle import dbsa_oracle as O

    meta, _ = load(name)
    c = oracle_cfg(meta)
    w = O.init_random(c, meta["spec"]["weight_seed"])
    t = meta["spec"]["task"]
    pool, tests, labels = O.recall_task(t["n_demos"], t["n_tests"], t["n_labels"], t["seed"])
    m = method(meta)
    part, kv, attended, index, refs, counts = O.encode_pool(
        c, w, pool, m["block_size"], m["seed"], "sink-prev-self", m["local_blocks"], m["granularity"])
    return dict(cfg=c, weights=w, pool=pool, tests=tests, labels=labels, partition=part, kv=kv,
                attended=attended, index=index, refs=refs, counts=counts, method=m)
