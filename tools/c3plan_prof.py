"""Host planning time of a C3 batch (64 queries) and the answer_stream pipeline:
per-batch host phases (select wait, plan, scorer, graph lookup, replay enqueue)."""
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
B = 64
batches = [([rng.integers(3, 1000, 32).tolist() for _ in range(B)], rng.random((B, 60))) for _ in range(12)]
for q, sc in batches[:2]:
    sess.answer(sc, q)
torch.cuda.synchronize()
t = {"select": 0.0, "plan": 0.0, "scorer": 0.0}
for q, sc in batches[2:6]:
    a = time.perf_counter(); ids = sess.select(sc); b = time.perf_counter()
    jobs, plan = sess.plan(ids, q); c = time.perf_counter()
    scorer = engine.LabelScorer(dm, plan, jobs, 4); d = time.perf_counter()
    t["select"] += b - a; t["plan"] += c - b; t["scorer"] += d - c
print({k: round(v / 4 * 1e3, 2) for k, v in t.items()}, "ms per 64-query batch")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
w0 = time.perf_counter(); e0.record()
n = 0
for _ in sess.answer_stream([(sc, q) for q, sc in batches[2:]]):
    n += 1
e1.record(); torch.cuda.synchronize()
print("answer_stream", n, "batches:", round(e0.elapsed_time(e1) / n, 2), "ms/batch (events),",
      round((time.perf_counter() - w0) * 1e3 / n, 2), "ms/batch wall")
g = next(iter(sess._graphs.values())) if hasattr(sess, "_graphs") and sess._graphs else None
print("graphs cached:", len(getattr(sess, "_graphs", {}) or {}))
# device-only: the same batches' graph replays, plans prepared up front
pre = []
for q, sc in batches[2:]:
    ids = sess.select(sc)
    jobs, plan = sess.plan(ids, q)
    scorer = engine.LabelScorer(dm, plan, jobs, 4)
    pre.append((jobs, plan, scorer))
torch.cuda.synchronize()
e0.record()
for jobs, plan, scorer in pre:
    g = sess._graph_for(jobs, plan, scorer)
    g.replay(plan, scorer)
e1.record(); torch.cuda.synchronize()
print("replay only:", round(e0.elapsed_time(e1) / len(pre), 2), "ms/batch")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in sess.answer_stream([(sc, q) for q, sc in batches[2:6]]):
        pass
    torch.cuda.synchronize()
ev = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
            if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0)
span = ev[-1][1] - ev[0][0]
gaps = []
end = ev[0][1]
for a, b, n in ev[1:]:
    if a - end > 50:
        gaps.append((round(a - end), n[:40]))
    end = max(end, b)
print("answer_stream 4 batches: span us", round(span), "gaps > 50us:", gaps[:20])
