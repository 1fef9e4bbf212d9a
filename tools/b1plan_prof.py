"""cProfile of the host planning of batch-1 Stage2Session.answer calls (C3 shape)."""
import cProfile, os, pstats, sys
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
qs = [([rng.integers(3, 1000, 32).tolist()], rng.random((1, 60))) for _ in range(40)]
for q, sc in qs[:5]:
    sess.answer(sc, q)[2].cpu()
pr = cProfile.Profile()
for q, sc in qs[5:]:
    pr.enable()
    ids = sess.select(sc)
    jobs, plan = sess.plan(ids, q)
    scorer = engine.LabelScorer(dm, plan, jobs, 4)
    pr.disable()
    sess.answer(sc, q)[2].cpu()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
