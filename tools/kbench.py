"""Kernel-only microbenchmark of K1 (stage-1) and K3 (stage-2) at the
Llama-3.1-8B / 90k-pool shapes, ONE layer, random K/V pages.  Used for ncu
captures (short) and quick A/B of kernel changes.

  python tools/kbench.py [--stage 1|2|both] [--batch 64] [--reps 5]
"""
import argparse, os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2503_08640_b200 as P
from paper_2503_08640_b200 import engine, masks, ops

ap = argparse.ArgumentParser()
ap.add_argument("--stage", default="both")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--ratio", type=float, default=0.3)
ap.add_argument("--groups", type=int, default=60)
ap.add_argument("--gtok", type=int, default=1500)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--target", type=int, default=0)
ap.add_argument("--order", default="query")
ap.add_argument("--schedule", default=None, help="chunk | query (default: by batch size)")
ap.add_argument("--chunk-m", type=int, default=2, help="M tiles per chunk-major work")
ap.add_argument("--dense", action="store_true", help="one contiguous T' chunk per query")
ap.add_argument("--dense-split", type=int, default=1, help="with --dense: the T' run as this many contiguous chunks")
args = ap.parse_args()

dev = torch.device("cuda", 0)
cfg = P.ModelConfig(d_model=args.heads * 128, n_layers=1, n_heads=args.heads, n_kv_heads=args.hkv, head_dim=128,
                    ffn_dim=14336, vocab_size=128256, rope_theta=500000.0, max_seq_len=131072)
rope = ops.rope_table(cfg.max_seq_len, 128, cfg.rope_theta, dev)


class _DM:  # the two attributes the plans read, plus the rope table
    config, device = cfg, dev

    def rope_for(self, rows):
        global rope
        if rows > rope.shape[0]:
            rope = ops.rope_table(rows, 128, cfg.rope_theta, dev)
        return rope


dm = _DM()
cache = P.SegmentedKVCache(cfg, dev, capacity_tokens=args.groups * args.gtok)
new = cache._reserve([args.gtok] * args.groups, [b"\0" * 32] * args.groups, [()] * args.groups)
g = torch.Generator(device=dev).manual_seed(0)
cache.store.k.normal_(generator=g)
cache.store.v.normal_(generator=g)
st = cache.store
qw = cfg.n_heads * 128
stride = qw + 2 * cfg.n_kv_heads * 128
hbm = 6537.3

def timeit(fn, reps):
    fn(); torch.cuda.synchronize()
    if os.environ.get("KB_GRAPH"):  # back-to-back launches in one CUDA graph: no host launch gaps
        n = 20
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(n):
                    fn()
        torch.cuda.current_stream().wait_stream(s)
        g.replay(); torch.cuda.synchronize()
        ts = []
        for _ in range(max(reps, 3)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / n)
        return float(np.median(ts))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in ev]))

if args.stage in ("1", "both"):
    plan = engine.Stage1Plan(dm, cache, new, masks.AttentionPattern.sink_prev_self(2))
    T = plan.n_tok
    qkv = torch.randn(T, stride, device=dev).to(torch.bfloat16)
    out = torch.empty(T, qw, dtype=torch.bfloat16, device=dev)
    def k1():
        ops.attention(q=qkv, q_tok_stride=stride, tok_pos=plan.pos, tok_lo=None, rope=rope,
                      pool=st.planes(), aux=None, n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads, head_dim=128,
                      works_dev=plan.works, n_works=plan.n_works, segs_dev=plan.segs_ptr(0), num_m=plan.num_m,
                      out=out, out_tok_stride=qw)
    ms = timeit(k1, args.reps)
    fl = plan.pairs * 4 * 128 * cfg.n_heads
    print(f"K1: {plan.n_works} works, {ms:.3f} ms, {fl/ms/1e9:.1f} TFLOP/s ({fl/ms/1e9/1701.9*100:.1f}% of 1701.9)", flush=True)

if args.stage in ("2", "both"):
    rng = np.random.default_rng(1)
    sess = P.Stage2Session(dm, cache,
                           [(b, 0, args.gtok) for b in range(args.groups)], [[5, 6, 7, 8]] * 4, args.ratio, "in-order")
    B = args.batch
    scores = rng.random((B, args.groups))
    ids = np.stack([[0] + sorted(rng.choice(np.arange(1, args.groups), sess.budget - 1, replace=False).tolist())
                    for _ in range(B)])
    q = [rng.integers(3, 1000, 32).tolist() for _ in range(B)]
    tabs, n_ctx = sess.chunks_for(ids)
    if args.dense:  # one contiguous run of T' pool rows per query (the dense comparator)
        Tp = int(n_ctx[0])
        k = args.dense_split
        cuts = [Tp * i // k for i in range(k + 1)]
        tabs = np.array([[[cuts[i], cuts[i + 1] - cuts[i], 0] for i in range(k)]] * B, np.int64)
    jobs = [engine.label_job(tabs[i], int(n_ctx[i]), q[i], sess.label_ids) for i in range(B)]
    plan = engine.Stage2Plan(dm, jobs, args.target or None, args.order, schedule=args.schedule)
    if plan.schedule == "chunk" and args.chunk_m != 2:
        plan.sched = engine.ChunkMajorSchedule(dm, jobs, plan.new, num_m=args.chunk_m)
        for name in ("works", "n_works", "n_merge", "merges", "max_rows"):
            setattr(plan, name, getattr(plan.sched, name))
    qkv = torch.randn(plan.n_tok, stride, device=dev).to(torch.bfloat16)
    out = torch.empty(plan.n_tok, qw, dtype=torch.bfloat16, device=dev)
    aux = (plan.k_aux, plan.v_aux, plan.aux_rows, 1)
    def k3():
        plan.sched.launch(dm, plan.new, 0, qkv, out, st.planes())
    def k3m():
        if plan.n_merge:
            ops.lse_merge(plan.part_o, plan.part_lse, plan.merges, plan.n_merge, plan.max_rows, cfg.n_heads,
                          cfg.n_kv_heads, 128, out, qw)
    ms = timeit(k3, args.reps)
    mm = timeit(k3m, args.reps)
    by = plan.kv_tokens * 2 * cfg.n_kv_heads * 128 * 2 + 2 * plan.n_tok * qw * 2
    print(f"K3 [{plan.schedule}]: B={B} {plan.n_works} works num_m={plan.sched.num_m if hasattr(plan.sched, 'num_m') else plan.num_m}, {ms:.3f} ms, {by/ms/1e6:.1f} GB/s "
          f"({by/ms/1e6/hbm*100:.1f}% of {hbm}); merge {mm:.3f} ms ({plan.n_merge} groups)", flush=True)
