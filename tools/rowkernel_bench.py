"""Per-launch time of the row kernels (SiLU*RMS-scale, RoPE+page store) at
decode (64 rows) and mixed-step (680 rows) sizes, C2 shape, CUDA events over
100 back-to-back launches (interleaved with a 1-row GEMM-like gap filler)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_16784_b200 import _lib as L  # noqa: E402

st = torch.cuda.current_stream().cuda_stream
res = {}
for T in (64, 680):
    u = torch.randn(T, 12288, device="cuda").to(torch.bfloat16)
    h = torch.randn(T, 4096, device="cuda").to(torch.bfloat16)
    qkv = torch.randn(T, 6144, device="cuda").to(torch.bfloat16)
    q = torch.empty(T, 4096, device="cuda", dtype=torch.bfloat16)
    kp = torch.zeros(4096, 8, 128, device="cuda", dtype=torch.bfloat16)
    vp = torch.zeros_like(kp)
    pos = torch.arange(T, dtype=torch.int32, device="cuda")
    pages = torch.arange(T, dtype=torch.int32, device="cuda")
    cos = torch.randn(40960, 64, device="cuda")
    sin = torch.randn(40960, 64, device="cuda")

    def silu():
        L.call("tim_silu_rms", u.data_ptr(), T, 12288, h.data_ptr(), 4096, 1e-6, L.DTYPE_BF16, st)

    def rope():
        L.call("tim_rope_kv_store", qkv.data_ptr(), h.data_ptr(), 4096, 1e-6, T, pos.data_ptr(),
               pages.data_ptr(), cos.data_ptr(), sin.data_ptr(), 32, 8, 128, q.data_ptr(),
               kp.data_ptr(), vp.data_ptr(), L.DTYPE_BF16, st)

    for name, fn in (("silu", silu), ("rope", rope)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[f"{name}_{T}_us"] = round(e0.elapsed_time(e1) * 10, 2)
print(json.dumps(res))
