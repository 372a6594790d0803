"""cuBLAS bf16 GEMM time at the decode shapes (weights streamed from HBM)."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = False
shapes = {"qkv": (4096, 6144), "wo": (4096, 4096), "w1": (4096, 12288), "w2": (12288, 4096)}
L = 36
res = {}
for M in (64, 128, 256):
    for name, (K, N) in shapes.items():
        Ws = [torch.randn(K, N, device="cuda", dtype=torch.bfloat16) for _ in range(8)]
        x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        for W in Ws:
            torch.matmul(x, W, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(40):
            if name in ("wo", "w2"):
                out.addmm_(x, Ws[i % 8]) if out.shape[1] == N else None
            else:
                torch.matmul(x, Ws[i % 8], out=out)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / 40
        res[f"M{M}_{name}"] = {"us": round(us, 2), "gbs": round(K * N * 2 / us / 1e3, 1)}
print(json.dumps(res, indent=0))
