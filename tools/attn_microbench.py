"""Decode-attention microbenchmark at the C2 shape (ncu target and quick A/B).

64 requests x L retained pages (default 724, the reference's C2 mean live),
Qwen3-8B GQA 32q/8kv, D=128, bf16, one layer.  Prints achieved algorithmic
GB/s from CUDA events (inputs > L2 by rotating over several layers' pools).
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_16784_b200 import _lib as L  # noqa: E402
from paper_2507_16784_b200.stepdesc import StepDesc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--live", type=int, default=724)
    ap.add_argument("--jitter", type=float, default=0.5)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--dump", action="store_true")
    ap.add_argument("--no-plan", action="store_true", help="skip tim_attn_plan (K1 searches itself)")
    ap.add_argument("--isolated", action="store_true",
                    help="CUDA events around every launch (as bench.py times layer 0): no PDL overlap")
    a = ap.parse_args()
    hq, hkv, d = 32, 8, 128
    rng = np.random.default_rng(0)
    lens = np.maximum(1, (a.live * (1 + a.jitter * (rng.random(a.batch) * 2 - 1)))).astype(int)
    cap = int(lens.sum()) + 16
    stride = int(lens.max())
    K = torch.randn(a.layers, cap, hkv, d, device="cuda").to(torch.bfloat16)
    V = torch.randn(a.layers, cap, hkv, d, device="cuda").to(torch.bfloat16)
    perm = rng.permutation(cap)
    tab = np.zeros((a.batch, stride), np.int32)
    o = 0
    for i, n in enumerate(lens):
        tab[i, :n] = perm[o:o + n]
        o += n
    tab_d = torch.from_numpy(tab).cuda()
    sd = StepDesc()
    for i, n in enumerate(lens):
        sd.dec.append((i, i, int(n), 1, int(n) - 1, 0))
    sd.serial = 0 if a.no_plan else 1
    step = torch.from_numpy(sd.pack()).cuda()
    q = torch.randn(a.batch, hq, d, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    ctas = a.ctas or L.load().tim_sm_count()
    ws = torch.zeros(L.load().tim_decode_ws_floats(ctas, a.batch, hkv, d), device="cuda")
    cnt = torch.zeros(a.batch * 8, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    if not a.no_plan:   # the per-step plan the engine computes once per step
        L.call("tim_attn_plan", step.data_ptr(), tab_d.data_ptr(), stride, ctas, a.batch, d, ws.data_ptr(), st)

    def run(l):
        L.call("tim_attn_decode", step.data_ptr(), 0, q.data_ptr(), out.data_ptr(), K[l].data_ptr(),
               V[l].data_ptr(), tab_d.data_ptr(), stride, hq, hkv, d, 1 / np.sqrt(d), ws.data_ptr(),
               cnt.data_ptr(), ctas, a.batch, L.DTYPE_BF16, st)

    for l in range(a.layers):
        run(l)
    torch.cuda.synchronize()
    # back-to-back launches over rotating layers (inputs > L2), so host launch
    # latency is hidden behind the previous kernel and events time the GPU only
    times = []
    if a.isolated:
        for it in range(a.iters):
            for l in range(a.layers):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run(l)
                e1.record()
                times.append((e0, e1))
        torch.cuda.synchronize()
        times = [x.elapsed_time(y) for x, y in times]
    for it in range(0 if a.isolated else a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for l in range(a.layers):
            run(l)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / a.layers)
    if a.trace:
        tr = torch.zeros(ctas * 8, dtype=torch.int64, device="cuda")
        L.call("tim_set_trace", tr.data_ptr())
        run(0)
        torch.cuda.synchronize()
        L.call("tim_set_trace", None)
        t = tr.view(-1, 8).cpu().numpy().astype(np.float64)
        t0 = t[:, 0].min()
        t = np.where(t > 0, (t - t0) / 1000.0, np.nan)   # unstamped slots -> nan
        print(json.dumps({k: [round(float(np.nanpercentile(t[:, i], p)), 2) if np.isfinite(t[:, i]).any() else None for p in (0, 50, 100)]
                          for i, k in enumerate(["start", "first", "loop_end", "end", "p_tile", "p_ids",
                                                 "pub_rel", "merge_ok"])}))
        if a.dump:
            pre = np.concatenate([[0], np.cumsum(lens)])
            N = int(pre[-1])
            for c in range(ctas):
                s0, s1 = c * N // ctas, (c + 1) * N // ctas
                nseg = int(np.searchsorted(pre, s1, side="left") - np.searchsorted(pre, s0, side="right") + 1)
                print(c, nseg, " ".join(f"{x:7.2f}" for x in t[c]))
    byts = int(lens.sum()) * hkv * d * 2 * 2 + a.batch * hq * d * 2 * 2
    ms = float(np.median(times))
    print(json.dumps({"tokens": int(lens.sum()), "bytes": byts, "ms": ms,
                      "gbs": byts / ms / 1e6, "ctas": ctas}))


if __name__ == "__main__":
    main()
