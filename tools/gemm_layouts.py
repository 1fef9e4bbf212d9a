"""Skinny-M GEMM layouts at the batch-1 shapes: x[M, K] @ W with W stored
[K, N] (the engine's layout) vs W^T stored [N, K] (nn.Linear layout), bf16
and fp32 output.  32 distinct weights per shape so the weights stream from
HBM as in the 32-layer forward; timed as one CUDA graph."""
import sys, torch
M = int(sys.argv[1]) if len(sys.argv) > 1 else 44
dev = torch.device("cuda")
shapes = [(4096, 6144, "qkv"), (4096, 4096, "o"), (4096, 28672, "gate_up"), (14336, 4096, "down")]
L = 16
for K, N, name in shapes:
    x = torch.randn(M, K, device=dev).to(torch.bfloat16)
    Ws = [torch.randn(K, N, device=dev).to(torch.bfloat16) for _ in range(L)]
    Wts = [w.t().contiguous() for w in Ws]
    res = {}
    for tag, fn in [("KN bf16", lambda i: torch.mm(x, Ws[i])),
                    ("NK bf16", lambda i: torch.mm(x, Wts[i].t())),
                    ("KN f32", lambda i: torch.mm(x, Ws[i], out_dtype=torch.float32)),
                    ("NK f32", lambda i: torch.mm(x, Wts[i].t(), out_dtype=torch.float32))]:
        for i in range(L):
            fn(i)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(L):
                fn(i)
        g.replay(); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); g.replay(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1000 / L)
        us = sorted(ts)[2]
        res[tag] = f"{us:6.1f} us {K * N * 2 / us / 1e6:5.2f} TB/s"
    print(name, M, " | ".join(f"{k}: {v}" for k, v in res.items()), flush=True)
    del Ws, Wts
