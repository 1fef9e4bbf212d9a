"""Batch-1 stage-2 latency at the C3 shape on random pages (no stage 1):
graph replays of single queries, for launch lists (ncu) and event timing."""
import os, sys
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
g = torch.Generator(device=dev).manual_seed(0)
cache.store.k.normal_(generator=g)
cache.store.v.normal_(generator=g)
cache.seal()
rng = np.random.default_rng(1)
labels = [rng.integers(3, 1000, 4).tolist() for _ in range(4)]
sess = P.Stage2Session(dm, cache, [(b, 0, 1500) for b in range(60)], labels, 0.3, "in-order")
q = [rng.integers(3, 1000, 32).tolist()]
sc = rng.random((1, 60))
ids = sess.select(sc)
jobs, plan = sess.plan(ids, q)
gr = engine.GraphedStage2(dm, cache.store, jobs, plan, 4)
scorer = engine.LabelScorer(dm, plan, jobs, 4)
ts = []
for i in range(int(os.environ.get("REPS", "10"))):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); gr.replay(plan, scorer); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print("batch-1 device ms:", np.median(ts[2:]) if len(ts) > 3 else ts, "works", plan.sched.n_works, plan.schedule)
