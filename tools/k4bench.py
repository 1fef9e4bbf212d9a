"""K4 (top-k group / example selection) at example granularity: 64 queries x
n units (e.g. 3,000 demonstrations of a 90k pool) at 30 % retrieval.

  python tools/k4bench.py [--units 3000] [--batch 64]
"""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2503_08640_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--units", type=int, nargs="+", default=[60, 1000, 3000, 25000])
ap.add_argument("--batch", type=int, default=64)
a = ap.parse_args()
for n in a.units:
    sc = torch.from_numpy(np.random.default_rng(0).random((a.batch, n))).cuda()
    for ordering in ("in-order", "low-to-high"):
        b = math.ceil(0.3 * n)
        ops.topk_select(sc, b, ordering); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ops.topk_select(sc, b, ordering)
        e1.record(); torch.cuda.synchronize()
        print(f"K4 n={n} budget={b} {ordering}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per batch of {a.batch}")
