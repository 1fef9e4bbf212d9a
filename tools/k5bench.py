"""K5 (fused label scoring) vs the unfused path it replaced (cuBLAS fp32
logits + one-pass log-prob gather), at the C3 batch shape: 832 distinct
scored rows x Llama-3 vocab 128,256, d 4096, 1,024 scored pairs.

  python tools/k5bench.py [--rows 832] [--reps 20]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_08640_b200 import ops

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=832)
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--vocab", type=int, default=128256)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
dev = torch.device("cuda", 0)
x = torch.randn(a.rows, a.d, device=dev).to(torch.bfloat16)
w = (torch.rand(a.vocab, a.d, device=dev) * 2 - 1).mul(1 / a.d ** 0.5).to(torch.bfloat16)
n_pairs = a.rows * 16 // 13
pr = torch.randint(0, a.rows, (n_pairs,), device=dev)
pt = torch.randint(0, a.vocab, (n_pairs,), device=dev).to(torch.int32)
ws = torch.empty(ops.label_score_workspace_shape(a.rows, a.vocab), dtype=torch.float32, device=dev)
out = torch.empty(n_pairs, dtype=torch.float32, device=dev)


def fused():
    ops.label_score(x, w, pr, pt, workspace=ws, out=out)


def unfused():
    logits = torch.mm(x.index_select(0, pr), w.t(), out_dtype=torch.float32)
    ops.label_logprob(logits, pt)


def t(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


tf, tu = t(fused), t(unfused)
fl = 2.0 * a.rows * a.d * a.vocab
print(f"K5 fused: {tf:.3f} ms ({fl / tf / 1e9:.0f} TFLOP/s over {a.rows} rows); "
      f"unfused (cuBLAS fp32 logits over {n_pairs} pair rows + log-prob): {tu:.3f} ms")
