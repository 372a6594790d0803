"""Per-CTA timeline of the layer-0 decode attention launch IN the bench's
context (C2 trajectory, a decode-only step): after the step ran, its pre graph
(plan, embed, layer-0 QKV GEMM, RoPE/store) is replayed and the attention
launch is re-issued between CUDA events with the per-CTA %globaltimer trace on
(start, first data, loop end, end, ...; 256-512 ns timer granularity).
Compare with tools/attn_microbench.py --trace --isolated.
usage: python tools/decode_trace_insitu.py [--step-frac 0.5]"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2507_16784_b200 import _lib as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--step-frac", type=float, default=0.5)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    eng, cfg, model = bench.build_engine(0, 64, 2)
    rt = eng.runtime
    rt.precapture()
    rt.recording = []
    while not eng.all_terminal():
        eng.step()
    records, rt.recording = rt.recording, None
    resident = rt.replay_upload(records)
    target = int(len(resident) * a.step_frac)
    while records[target][0].ext or records[target][0].n_rows != 64:
        target += 1
    for i, (sd, step, fw) in enumerate(resident[: target + 1]):
        rt._execute(sd, step, fw)
    sd, step, fw = resident[target]
    torch.cuda.synchronize()
    key = (sd.rows_pad, False)
    g = rt.graphs[key]
    times = []
    tr = torch.zeros(rt.sms * 8, dtype=torch.int64, device="cuda")
    for rep in range(a.reps):
        g["pre"].replay()
        if rep == a.reps - 1:
            L.call("tim_set_trace", tr.data_ptr())
        ev = []
        model._attn(rt, rt.gstep.data_ptr(), 0, sd.rows_pad, False, ev)
        torch.cuda.synchronize()
        times.append(ev[0][0].elapsed_time(ev[0][1]) * 1e3)
    L.call("tim_set_trace", None)
    t = tr.view(-1, 8).cpu().numpy().astype(np.float64)
    t0 = t[:, 0][t[:, 0] > 0].min()
    t = np.where(t > 0, (t - t0) / 1000.0, np.nan)
    keys = ["start", "first", "loop_end", "end", "p_tile", "p_ids", "pub_rel", "merge_ok"]
    print(json.dumps({k: [round(float(np.nanpercentile(t[:, i], p)), 2) if np.isfinite(t[:, i]).any() else None
                          for p in (0, 50, 100)] for i, k in enumerate(keys)}))
    kv = sum(sg[1] + sg[2] for sg in sd.segs)
    byts = kv * cfg.n_kv * cfg.head_dim * 4 + sd.n_rows * cfg.heads * cfg.head_dim * 4
    us = float(np.median(times[2:]))
    print(json.dumps({"step": target, "kv_tokens": kv, "bytes": byts, "us_events_median": us,
                      "gbs": byts / us / 1e3, "all_us": [round(x, 1) for x in times]}))


if __name__ == "__main__":
    main()
