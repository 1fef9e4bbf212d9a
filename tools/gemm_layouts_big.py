"""cuBLAS at large M (C3 batch 2816 tokens, stage-1 pool 22528-token chunk): W [K, N] vs W^T [N, K] (K-major)."""
import torch
dev = torch.device("cuda")
for M in (2816, 22528):
    for K, N, name in [(4096, 6144, "qkv"), (4096, 4096, "o"), (4096, 28672, "gate_up"), (14336, 4096, "down")]:
        x = torch.randn(M, K, device=dev).to(torch.bfloat16)
        W = torch.randn(K, N, device=dev).to(torch.bfloat16)
        Wt = W.t().contiguous()
        res = []
        for tag, fn in [("KN", lambda: torch.mm(x, W)), ("NK", lambda: torch.mm(x, Wt.t())),
                        ("KN f32", lambda: torch.mm(x, W, out_dtype=torch.float32)),
                        ("NK f32", lambda: torch.mm(x, Wt.t(), out_dtype=torch.float32))]:
            for _ in range(3): fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10): fn()
            b.record(); torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 10
            res.append(f"{tag}: {ms*1000:7.1f} us {2*M*N*K/ms/1e9:6.0f} TF/s")
        print(M, name, " | ".join(res), flush=True)
