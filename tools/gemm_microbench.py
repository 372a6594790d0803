"""cuBLAS bf16 GEMM time at the decode shapes (weights streamed from HBM).

Times the four per-layer GEMMs of the Qwen3-8B-shaped model exactly as the
forward issues them (matmul into a buffer for qkv / w1, addmm_ residual for
wo / w2), rotating over 8 weight copies so the weights come from HBM.
"""
import json
import os
import sys

import torch

torch.backends.cuda.matmul.allow_tf32 = False
lib = sys.argv[1] if len(sys.argv) > 1 else "default"
if lib in ("cublas", "cublaslt"):
    torch.backends.cuda.preferred_blas_library(lib)
shapes = {"qkv": (4096, 6144, False), "wo": (4096, 4096, True), "w1": (4096, 12288, False),
          "w2": (12288, 4096, True)}
res = {"lib": lib, "env_DISABLE_ADDMM_CUDA_LT": os.environ.get("DISABLE_ADDMM_CUDA_LT")}
tot = {}
for M in (64, 128, 256):
    tot[M] = 0.0
    for name, (K, N, resid) in shapes.items():
        Ws = [torch.randn(K, N, device="cuda", dtype=torch.bfloat16) for _ in range(8)]
        x = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)

        def run(i):
            if resid:
                out.addmm_(x, Ws[i % 8])
            else:
                torch.matmul(x, Ws[i % 8], out=out)

        for i in range(8):
            run(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(48):
            run(i)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / 48
        tot[M] += us
        res[f"M{M}_{name}"] = {"us": round(us, 2), "gbs": round(K * N * 2 / us / 1e3, 1)}
    res[f"M{M}_layer_us"] = round(tot[M], 2)
print(json.dumps(res))
