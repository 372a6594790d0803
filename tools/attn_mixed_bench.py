"""Mixed decode + re-encode attention step at the C2 shape: 64 decode queries
(retained ~724) plus E re-encode segments of n rows over an m-token prefix.
Variants: all rows as 4-query decode tiles (mode 0), or the multi-token rows
as mode-1 tiles (tcgen05 kernel: 32 queries x one kv head).  Prints median us and unique-byte GB/s per variant."""
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
    ap.add_argument("--ext", type=int, default=6)
    ap.add_argument("--n", type=int, default=150)
    ap.add_argument("--m", type=int, default=600)
    ap.add_argument("--layers", type=int, default=6)
    ap.add_argument("--only", default="")
    ap.add_argument("--trace", action="store_true")
    a = ap.parse_args()
    hq, hkv, d, B = 32, 8, 128, 64
    rng = np.random.default_rng(0)
    lens = np.maximum(1, (724 * (1 + 0.5 * (rng.random(B) * 2 - 1)))).astype(int)
    segs = [(int(L_ - 1), 1) for L_ in lens] + [(a.m, a.n)] * a.ext     # (m, n) per request
    tot = sum(m + n for m, n in segs)
    cap = tot + 16
    stride = max(m + n for m, n in segs)
    K = torch.randn(a.layers, cap, hkv, d, device="cuda").to(torch.bfloat16)
    V = torch.randn(a.layers, cap, hkv, d, device="cuda").to(torch.bfloat16)
    perm = rng.permutation(cap)
    tab = np.zeros((len(segs), stride), np.int32)
    o = 0
    for i, (m, n) in enumerate(segs):
        tab[i, :m + n] = perm[o:o + m + n]
        o += m + n
    tab_d = torch.from_numpy(tab).cuda()
    rows = sum(n for _, n in segs)
    q = torch.randn(rows, hq, d, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    ctas = L.load().tim_sm_count()
    st = torch.cuda.current_stream().cuda_stream
    ub = tot * hkv * d * 4 + rows * hq * d * 4
    res = {}
    qpi = L.load().tim_extend_queries_per_item(hq, hkv, d, L.DTYPE_BF16)
    ngroups = L.load().tim_extend_head_groups(hq, hkv, d)
    for variant, (qpt, ngr) in {"mode0": (4, 1), "mode1": (qpi, ngroups), "mode2": (qpi, ngroups)}.items():
        if a.only and variant != a.only:
            continue
        sd = StepDesc()
        row = 0
        for i, (m, n) in enumerate(segs):
            if n == 1 or variant == "mode0":
                for q0 in range(0, n, 4):
                    nq = min(4, n - q0)
                    sd.dec.append((row + q0, i, m + q0 + nq, nq, m, 0))
            else:
                for q0 in range(0, n, qpt):
                    nq = min(qpt, n - q0)
                    for g in range(ngr):
                        sd.ext.append((row + q0, i, m + q0 + nq, nq, m, g))
            row += n
        sd.ctas = ctas
        step = torch.from_numpy(sd.pack()).cuda()
        split = (sd.offsets["split_dec_ctas"], sd.offsets["split_ext_ctas"])
        maxd = max(len(sd.dec), len(sd.ext)) + 8
        ws = torch.zeros(L.load().tim_decode_ws_floats(ctas, maxd, hkv, d), device="cuda")
        cnt = torch.zeros(maxd * 8, dtype=torch.int32, device="cuda")

        def run(l):
            if variant == "mode2":
                L.call("tim_attn_decode", step.data_ptr(), 2, q.data_ptr(), out.data_ptr(), K[l].data_ptr(),
                       V[l].data_ptr(), tab_d.data_ptr(), stride, hq, hkv, d, 1 / np.sqrt(d), ws.data_ptr(),
                       cnt.data_ptr(), ctas, maxd, L.DTYPE_BF16, st)
                return
            L.call("tim_attn_decode", step.data_ptr(), 0, q.data_ptr(), out.data_ptr(), K[l].data_ptr(),
                   V[l].data_ptr(), tab_d.data_ptr(), stride, hq, hkv, d, 1 / np.sqrt(d), ws.data_ptr(),
                   cnt.data_ptr(), ctas, maxd, L.DTYPE_BF16, st)
            if sd.ext:
                L.call("tim_attn_decode", step.data_ptr(), 1, q.data_ptr(),
                       out.data_ptr(), K[l].data_ptr(), V[l].data_ptr(), tab_d.data_ptr(), stride, hq, hkv,
                       d, 1 / np.sqrt(d), ws.data_ptr(), cnt.data_ptr(), ctas, maxd, L.DTYPE_BF16, st)

        for l in range(a.layers):
            run(l)
        torch.cuda.synchronize()
        ref = out.float().clone()
        times = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for l in range(a.layers):
                run(l)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1000 / a.layers)
        us = float(np.median(times))
        if a.trace and variant == "mode2":
            ctas = L.load().tim_sm_count()
            tr = torch.zeros(ctas * 8, dtype=torch.int64, device="cuda")
            L.call("tim_set_trace", tr.data_ptr())
            run(0)
            torch.cuda.synchronize()
            L.call("tim_set_trace", None)
            t = tr.view(ctas, 8).cpu().numpy().astype(np.float64)
            t0 = t[:, 0][t[:, 0] > 0].min()
            dec, ext = t[:split[0]], t[split[0]:split[0] + split[1]]
            pct = lambda x: [round(float(np.percentile((x - t0) / 1000, p)), 2) for p in (0, 50, 90, 100)]
            print(json.dumps({"dec_end": pct(dec[:, 3]), "dec_loop_end": pct(dec[:, 2]), "ext_end": pct(ext[:, 3])}),
                  file=sys.stderr)
        if a.trace and sd.ext:
            tr = torch.zeros(64 * 8, dtype=torch.int64, device="cuda")
            L.call("tim_tc_trace", tr.data_ptr())
            run(0)
            torch.cuda.synchronize()
            L.call("tim_tc_trace", None)
            t = tr.view(64, 8).cpu().numpy().astype(np.float64)
            t0 = t[t > 0].min()
            names = ["prod_slot_free", "pv1_issue", "s0_issue", "pv0_issue", "sm0_s_ready", "sm0_p_done",
                     "sm1_s_ready", "sm1_p_done"]
            for g in range(64):
                if t[g, 0] == 0:
                    break
                print(g, " ".join(f"{n}={(t[g, i] - t0) / 1000:7.2f}" for i, n in enumerate(names)), file=sys.stderr)
        res[variant] = {"us": round(us, 1), "split": split, "gbs": round(ub / us / 1e3), "tiles": len(sd.dec) + len(sd.ext),
                        "streamed_tokens": int(sum(t[2] for t in sd.dec) + sum(t[2] for t in sd.ext) / ngr)}
        res.setdefault("_outs", []).append(ref)
    outs = res.pop("_outs")
    if len(outs) == 3:
        res["maxdiff_mode1_vs_0"] = float((outs[1] - outs[0]).abs().max())
        res["maxdiff_mode2_vs_0"] = float((outs[2] - outs[0]).abs().max())
    res["unique_MB"] = round(ub / 1e6, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
