"""Run K2 (tcgen05 multi-token items, tim_attn_decode mode 1) alone on a small
ragged set of re-encode / extend segments and check it against a torch fp32
reference -- a sanitizer-friendly single-kernel workload (no decode tiles).
usage: compute-sanitizer --tool racecheck python tools/k2_only.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_16784_b200 import _lib as L  # noqa: E402
from paper_2507_16784_b200.stepdesc import StepDesc  # noqa: E402

hq, hkv, d = 32, 8, 128
segs = [(0, 40), (100, 64), (300, 150), (37, 9)]          # (prefix m, rows n)
rng = np.random.default_rng(0)
tot = sum(m + n for m, n in segs)
K = torch.randn(tot + 8, hkv, d, device="cuda").to(torch.bfloat16)
V = torch.randn(tot + 8, hkv, d, device="cuda").to(torch.bfloat16)
stride = max(m + n for m, n in segs)
perm = rng.permutation(tot + 8)
tab = np.zeros((len(segs), stride), np.int32)
o = 0
for i, (m, n) in enumerate(segs):
    tab[i, :m + n] = perm[o:o + m + n]
    o += m + n
tab_d = torch.from_numpy(tab).cuda()
rows = sum(n for _, n in segs)
q = torch.randn(rows, hq, d, device="cuda").to(torch.bfloat16)
out = torch.zeros_like(q)
qpi = L.load().tim_extend_queries_per_item(hq, hkv, d, L.DTYPE_BF16)
ngr = L.load().tim_extend_head_groups(hq, hkv, d)
sd = StepDesc()
row = 0
for i, (m, n) in enumerate(segs):
    for q0 in range(0, n, qpi):
        nq = min(qpi, n - q0)
        for g in range(ngr):
            sd.ext.append((row + q0, i, m + q0 + nq, nq, m, g))
    row += n
sd.ctas = L.load().tim_sm_count()
step = torch.from_numpy(sd.pack()).cuda()
ws = torch.zeros(L.load().tim_decode_ws_floats(sd.ctas, 64, hkv, d), device="cuda")
cnt = torch.zeros(64 * 8, dtype=torch.int32, device="cuda")
L.call("tim_attn_decode", step.data_ptr(), 1, q.data_ptr(), out.data_ptr(), K.data_ptr(), V.data_ptr(),
       tab_d.data_ptr(), stride, hq, hkv, d, 1 / np.sqrt(d), ws.data_ptr(), cnt.data_ptr(), sd.ctas, 64,
       L.DTYPE_BF16, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
worst, row = 0.0, 0
for i, (m, n) in enumerate(segs):
    pages = torch.from_numpy(tab[i, :m + n].astype(np.int64)).cuda()
    k, v = K[pages].float(), V[pages].float()                 # (m+n, hkv, d)
    qq = q[row:row + n].float().view(n, hkv, hq // hkv, d)
    s = torch.einsum("qhgd,khd->hgqk", qq, k) / np.sqrt(d)
    mask = torch.arange(m + n, device="cuda")[None, :] > (m + torch.arange(n, device="cuda"))[:, None]
    s = s.masked_fill(mask, float("-inf"))
    ref = torch.einsum("hgqk,khd->qhgd", torch.softmax(s, -1), v).reshape(n, hq, d)
    worst = max(worst, float((ref - out[row:row + n].float()).abs().max()))
    row += n
print(f"K2 alone: {len(sd.ext)} items, max |out - fp32 ref| = {worst:.4f}")
assert worst < 2e-2
