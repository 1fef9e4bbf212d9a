"""The sharded multi-GPU paths ACROSS PROCESSES on one B200: two ranks
(gloo over 127.0.0.1; device tensors are staged through host memory because
NCCL cannot run two ranks on one device) run the group-sharded stage 1 with
its per-layer halo exchange and the C5 stage 2 (per-rank chunk-major K3 +
per-rank K3m, all-gather, final K3m) on the C1 golden case
(tests/_mp_sharded_worker.py).  Every rank is checked against the
reference's goldens (tests/golden, made by the unmodified reference).
"""

import json
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from golden_util import load  # noqa: E402

HERE = Path(__file__).resolve().parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_paths_two_processes(tmp_path):
    world, port = 2, _free_port()
    outs = [tmp_path / f"rank{r}.json" for r in range(world)]
    procs = [subprocess.Popen([sys.executable, str(HERE / "_mp_sharded_worker.py"), str(r), str(world), str(port),
                               str(outs[r])], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=600)[0])
        except subprocess.TimeoutExpired:
            p.kill()
            logs.append(p.communicate()[0])
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-4000:]}"
    meta, a = load("c1")
    res = [json.loads(o.read_text()) for o in outs]
    for r in res:
        assert r["halo"] > 0  # the halo exchange actually crossed processes
        assert r["pairs"] == meta["attended_pairs"]
        assert r["page_err"] < 1e-2, r["page_err"]
        scores = np.asarray(r["scores"])
        for qi, q in enumerate(meta["queries"]):
            assert np.abs(scores[qi] - a[f"q{qi}_label_scores"]).max() < 0.04, (r["rank"], qi)
            assert r["labels"][qi] == q["predicted"], (r["rank"], qi)
    # both ranks computed the same answers (every rank runs the full forward)
    assert res[0]["labels"] == res[1]["labels"]
    assert np.abs(np.asarray(res[0]["scores"]) - np.asarray(res[1]["scores"])).max() < 1e-6
