"""Skinny decode GEMM (tim_gemm_skinny) vs a torch fp32 reference (GPU).

Tolerance: bf16 inputs, fp32 accumulation, bf16 output -> |y - ref| <= 1e-2 *
max|ref| + bf16 rounding of the output."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2507_16784_b200 import _lib as L

pytestmark = pytest.mark.gpu


def _tmap(t, box_rows=64):
    buf = (ctypes.c_uint8 * 128)()
    L.call("tim_tmap_2d_bf16", ctypes.addressof(buf), t.data_ptr(), t.shape[0], t.shape[1],
           box_rows, 64)
    return buf


@pytest.mark.parametrize("n,k", [(6144, 4096), (4096, 4096), (12288, 4096), (4096, 12288), (512, 256)])
@pytest.mark.parametrize("m", [64, 37, 1])
@pytest.mark.parametrize("ctas", [148, 7])
@pytest.mark.parametrize("residual", [False, True])
def test_skinny_gemm_matches_torch(n, k, m, ctas, residual):
    g = torch.Generator(device="cuda").manual_seed(n + k + m)
    x = (torch.randn(64, k, device="cuda", generator=g) * 0.5).to(torch.bfloat16)   # buffer of 64 rows
    wt = (torch.randn(n, k, device="cuda", generator=g) / np.sqrt(k)).to(torch.bfloat16)
    y = (torch.randn(64, n, device="cuda", generator=g)).to(torch.bfloat16)
    y0 = y.clone()
    ws = torch.zeros(L.load().tim_gemm_ws_floats(ctas, n), device="cuda")
    cnt = torch.zeros(n // 64, dtype=torch.int32, device="cuda")
    tx, tw = _tmap(x), _tmap(wt, 128)
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(2):   # counters self-reset
        y.copy_(y0)
        L.call("tim_gemm_skinny", ctypes.addressof(tx), ctypes.addressof(tw), y.data_ptr(),
               y.data_ptr() if residual else None, m, n, k, ws.data_ptr(), cnt.data_ptr(), ctas, st)
        torch.cuda.synchronize()
        assert int(cnt.abs().sum()) == 0
        ref = x[:m].float() @ wt.float().t() + (y0[:m].float() if residual else 0)
        got = y[:m].float()
        err = (got - ref).abs().max().item()
        assert err <= 1e-2 * ref.abs().max().item() + 0.02, err
        assert torch.equal(y[m:], y0[m:])   # rows past M untouched
