import sys, json
import numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2507_16784_b200 import _lib as L
from paper_2507_16784_b200.stepdesc import StepDesc
hq, hkv, d, B, live = 32, 8, 128, 64, 724
rng = np.random.default_rng(0)
lens = np.maximum(1, (live * (1 + 0.5 * (rng.random(B) * 2 - 1)))).astype(int)
cap = int(lens.sum()) + 16; stride = int(lens.max())
K = torch.randn(cap, hkv, d, device="cuda").to(torch.bfloat16); V = torch.randn(cap, hkv, d, device="cuda").to(torch.bfloat16)
perm = rng.permutation(cap); tab = np.zeros((B, stride), np.int32); o = 0
for i, n in enumerate(lens): tab[i, :n] = perm[o:o + n]; o += n
tab_d = torch.from_numpy(tab).cuda()
sd = StepDesc()
for i, n in enumerate(lens): sd.dec.append((i, i, int(n), 1, int(n) - 1, 0))
sd.serial = 1
step = torch.from_numpy(sd.pack()).cuda()
q = torch.randn(B, hq, d, device="cuda").to(torch.bfloat16); out = torch.empty_like(q)
ctas = L.load().tim_sm_count()
ws = torch.zeros(L.load().tim_decode_ws_floats(ctas, B, hkv, d), device="cuda")
cnt = torch.zeros(B * 8, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
L.call("tim_attn_plan", step.data_ptr(), tab_d.data_ptr(), stride, ctas, B, d, ws.data_ptr(), st)
run = lambda: L.call("tim_attn_decode", step.data_ptr(), 0, q.data_ptr(), out.data_ptr(), K.data_ptr(), V.data_ptr(), tab_d.data_ptr(), stride, hq, hkv, d, 1 / np.sqrt(d), ws.data_ptr(), cnt.data_ptr(), ctas, B, L.DTYPE_BF16, st)
for _ in range(5): run()
torch.cuda.synchronize()
tr = torch.zeros(ctas * 8, dtype=torch.int64, device="cuda")
L.call("tim_set_trace", tr.data_ptr())
torch.cuda._sleep(2000000); run(); torch.cuda.synchronize()
L.call("tim_set_trace", None)
t = tr.view(-1, 8).cpu().numpy()
t0 = t[:, 0].min()
end = (t[:, 3] - t0) / 1000.0; loop_end = (t[:, 2] - t0) / 1000.0
mg = t[:, 5] > 0
print("merger CTAs", mg.sum(), "of", ctas)
print("cycles: count-wait p50 %.0f max %.0f | merge p50 %.0f max %.0f | store+publish p50 %.0f max %.0f" % (
    np.median(t[mg, 4]), t[mg, 4].max(), np.median(t[mg, 5]), t[mg, 5].max(), np.median(t[mg, 6]), t[mg, 6].max()))
print("non-merger store+publish cycles p50 %.0f max %.0f" % (np.median(t[~mg, 6]), t[~mg, 6].max()))
slow = np.argsort(-end)[:6]
for i in slow: print(i, "merger" if mg[i] else "-", "loop_end %.2f end %.2f" % (loop_end[i], end[i]), "wait %d merge %d pub %d" % tuple(t[i, 4:7]))
