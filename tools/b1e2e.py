"""Host-side phases of a batch-1 Stage2Session.answer at the C3 shape (random pages)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_08640_b200 as P
from paper_2503_08640_b200 import engine

dev = torch.device("cuda", 0)
cfg = P.ModelConfig(d_model=4096, n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
                    vocab_size=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq_len=131072)
dm = engine.DeviceModel.random(cfg, 0, dev)
cache = P.SegmentedKVCache(cfg, dev, capacity_tokens=60 * 1500)
cache._reserve([1500] * 60, [b"\0" * 32] * 60, [()] * 60)
cache.seal()
rng = np.random.default_rng(1)
labels = [rng.integers(3, 1000, 4).tolist() for _ in range(4)]
sess = P.Stage2Session(dm, cache, [(b, 0, 1500) for b in range(60)], labels, 0.3, "in-order")
ph = {k: [] for k in ("select", "plan", "scorer+key", "replay", "d2h", "total")}
for it in range(12):
    q = [rng.integers(3, 1000, 32).tolist()]
    sc = rng.random((1, 60))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ids = sess.select(sc)
    t1 = time.perf_counter()
    jobs, plan = sess.plan(ids, q)
    t2 = time.perf_counter()
    scorer = engine.LabelScorer(dm, plan, jobs, 4)
    key = engine.plan_key(plan, scorer)
    graphs = sess.__dict__.setdefault("_graphs", {})
    if key not in graphs:
        graphs[key] = engine.GraphedStage2(dm, cache.store, jobs, plan, 4)
    t3 = time.perf_counter()
    s, best = graphs[key].replay(plan, scorer)
    t4 = time.perf_counter()
    best.cpu()
    t5 = time.perf_counter()
    if it >= 2:
        for k, v in zip(ph, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t5 - t0)):
            ph[k].append(v * 1e3)
print({k: round(float(np.median(v)), 3) for k, v in ph.items()})
