"""Per-CTA phase timeline of tim_gemm_skinny (globaltimer stamps, ns).

Phases: 0 start, 1 W prologue issued, 2 griddep wait done, 3 first stage full
(MMA), 4 last MMA commit, 5 last accumulator ready (epilogue), 6 epilogue end.
"""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_16784_b200 import _lib as L  # noqa: E402

lib = L.load()
sms = lib.tim_sm_count()
out = {}
raw = {}
for name, (n, k, resid) in {"qkv": (6144, 4096, False), "w2": (4096, 12288, True)}.items():
    wts = [torch.randn(n, k, device="cuda").to(torch.bfloat16) for _ in range(4)]
    x = torch.randn(64, k, device="cuda").to(torch.bfloat16)
    y = torch.zeros(64, n, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(lib.tim_gemm_ws_floats(sms, n), device="cuda")
    cnt = torch.zeros(n // 64, dtype=torch.int32, device="cuda")
    tx = (ctypes.c_uint8 * 128)()
    L.call("tim_tmap_2d_bf16", ctypes.addressof(tx), x.data_ptr(), 64, k, 64, 64)
    tws = []
    for w in wts:
        b = (ctypes.c_uint8 * 128)()
        L.call("tim_tmap_2d_bf16", ctypes.addressof(b), w.data_ptr(), n, k, 128, 64)
        tws.append(b)
    st = torch.cuda.current_stream().cuda_stream

    def run(i):
        L.call("tim_gemm_skinny", ctypes.addressof(tx), ctypes.addressof(tws[i % 4]), y.data_ptr(),
               y.data_ptr() if resid else None, 64, n, k, ws.data_ptr(), cnt.data_ptr(), sms, st)

    for i in range(6):
        run(i)
    torch.cuda.synchronize()
    for mode in ("isolated", "back_to_back"):
        if mode == "back_to_back":
            run(0)
        lib.tim_gemm_trace(1, None, 0)
        run(1)
        lib.tim_gemm_trace(0, None, 0)
        torch.cuda.synchronize()
        buf = (ctypes.c_uint64 * (160 * 16))()
        L.call("tim_gemm_trace", 0, buf, 160 * 16)
        t = np.array(buf, dtype=np.int64).reshape(160, 16)[:sms, :10]
        raw[f"{name}_{mode}"] = t.copy()
        t0 = t[:, 0].min()
        rel = (t - t0) / 1000.0
        out[f"{name}_{mode}"] = {
            f"p{i}": [round(float(np.min(rel[:, i])), 2), round(float(np.median(rel[:, i])), 2),
                      round(float(np.max(rel[:, i])), 2)] for i in range(8)}
print(json.dumps(out))
np.savez("gpurun_out/gemm_trace.npz", **raw)
