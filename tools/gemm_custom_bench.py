"""Per-layer decode GEMMs (M=64): tim_gemm_skinny vs cuBLAS (torch), weights from HBM."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_16784_b200 import _lib as L  # noqa: E402

shapes = {"qkv": (6144, 4096, False), "wo": (4096, 4096, True), "w1": (12288, 4096, False),
          "w2": (4096, 12288, True)}
sms = L.load().tim_sm_count()
out = {}
tot_c = tot_t = 0.0
for name, (n, k, resid) in shapes.items():
    wts = [torch.randn(n, k, device="cuda").to(torch.bfloat16) for _ in range(8)]
    x = torch.randn(64, k, device="cuda").to(torch.bfloat16)
    y = torch.zeros(64, n, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(L.load().tim_gemm_ws_floats(sms, n), device="cuda")
    cnt = torch.zeros(n // 64, dtype=torch.int32, device="cuda")
    tx = (ctypes.c_uint8 * 128)()
    L.call("tim_tmap_2d_bf16", ctypes.addressof(tx), x.data_ptr(), 64, k, 64, 64)
    tws = []
    for w in wts:
        b = (ctypes.c_uint8 * 128)()
        L.call("tim_tmap_2d_bf16", ctypes.addressof(b), w.data_ptr(), n, k, 128, 64)
        tws.append(b)
    st = torch.cuda.current_stream().cuda_stream

    def custom(i):
        L.call("tim_gemm_skinny", ctypes.addressof(tx), ctypes.addressof(tws[i % 8]), y.data_ptr(),
               y.data_ptr() if resid else None, 64, n, k, ws.data_ptr(), cnt.data_ptr(), sms, st)

    def cublas(i):
        if resid:
            y.addmm_(x, wts[i % 8].t())
        else:
            torch.matmul(x, wts[i % 8].t(), out=y)

    res = {}
    for tag, fn in (("custom", custom), ("cublas", cublas)):
        for i in range(8):
            fn(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(48):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / 48
        res[tag] = {"us": round(us, 2), "gbs": round(n * k * 2 / us / 1e3, 1)}
    tot_c += res["custom"]["us"]
    tot_t += res["cublas"]["us"]
    out[name] = res
out["layer_us"] = {"custom": round(tot_c, 2), "cublas": round(tot_t, 2)}
print(json.dumps(out))
