"""Stage-2 chunk-major K3 at the 8B shape (random pages, no stage 1): every
layer's launch of the padded schedule, synchronised, with table checks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_08640_b200 as P
from paper_2503_08640_b200 import engine, ops

dev = torch.device("cuda", 0)
L = int(os.environ.get("LAYERS", "32"))
cfg = P.ModelConfig(d_model=4096, n_layers=L, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
                    vocab_size=128256, rope_theta=500000.0, norm_eps=1e-5, max_seq_len=131072)


class _DM:
    config, device = cfg, dev
    rope = ops.rope_table(cfg.max_seq_len, 128, cfg.rope_theta, dev)

    def rope_for(self, rows):
        return self.rope


dm = _DM()
cache = P.SegmentedKVCache(cfg, dev, capacity_tokens=60 * 1500)
cache._reserve([1500] * 60, [b"\0" * 32] * 60, [()] * 60)
g = torch.Generator(device=dev).manual_seed(0)
cache.store.k.normal_(generator=g)
cache.store.v.normal_(generator=g)
cache.seal()
rng = np.random.default_rng(1)
labels = [rng.integers(3, 1000, 4).tolist() for _ in range(4)]
sess = P.Stage2Session(dm, cache, [(b, 0, 1500) for b in range(60)], labels, 0.3, "in-order")
q = [rng.integers(3, 1000, 32).tolist() for _ in range(64)]
ids = sess.select(rng.random((64, 60)))
jobs, plan = sess.plan(ids, q)
sc = plan.sched
n0, s0 = sc.n_works, sc.n_segs
segs_before = sc.segs.cpu().numpy().reshape(L, -1)
sc.pad_to(n0 + 500, s0 + 50)
segs_after = sc.segs.cpu().numpy().reshape(L, -1)
assert (segs_after[:, : s0 * 32] == segs_before).all(), "segs mismatch"
works = sc.works.cpu().numpy().view(ops.WORK_DTYPE)
print("works", n0, "->", sc.n_works, "segs", s0, "->", sc.n_segs, "max seg_end", works["seg_end"].max(), flush=True)
qw = 32 * 128
stride = qw + 2 * 8 * 128
qkv = torch.randn(plan.n_tok, stride, device=dev).to(torch.bfloat16)
out = torch.empty(plan.n_tok, qw, dtype=torch.bfloat16, device=dev)
for layer in range(L):
    sc.launch(dm, plan.new, layer, qkv, out, cache.store.planes())
    torch.cuda.synchronize()
    print("layer", layer, "ok", flush=True)
