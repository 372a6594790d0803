"""Probe: tim_gemm_skinny time for the o_proj shape with residual aliasing y,
a separate residual buffer, and no residual."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_16784_b200 import _lib as L  # noqa: E402

lib = L.load()
sms = lib.tim_sm_count()
n, k = 4096, 4096
wts = [torch.randn(n, k, device="cuda").to(torch.bfloat16) for _ in range(8)]
x = torch.randn(64, k, device="cuda").to(torch.bfloat16)
y = torch.zeros(64, n, device="cuda", dtype=torch.bfloat16)
r2 = torch.zeros(64, n, device="cuda", dtype=torch.bfloat16)
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
out = {}
for tag, res in (("none", None), ("alias", y.data_ptr()), ("separate", r2.data_ptr()), ("none2", None)):
    def run(i):
        L.call("tim_gemm_skinny", ctypes.addressof(tx), ctypes.addressof(tws[i % 8]), y.data_ptr(),
               res, 64, n, k, ws.data_ptr(), cnt.data_ptr(), sms, st)
    for i in range(8):
        run(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(48):
        run(i)
    e1.record()
    torch.cuda.synchronize()
    out[tag] = round(e0.elapsed_time(e1) * 1000 / 48, 2)
print(json.dumps(out))
