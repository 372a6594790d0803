"""Recalibrate the mode-2 split cost model (StepDesc._split_cost) on the bench's
own mixed steps.  Replays the C2 trajectory (bench.py's engine and stride
sampling); right after each sampled step that has multi-token rows, re-packs
that step's descriptor under each candidate (EXT_US_PER_ITEM,
EXT_US_PER_QBLOCK_BLOCK, DEC_US_PER_TOKEN) and times the layer-0 attention
launch (plan kernel outside the events, as in bench.py's pre-graph), CUDA
events around each launch.  Prints mean us per candidate.
usage: python tools/split_sweep.py [--steps 200]"""
import argparse
import itertools
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2507_16784_b200 import _lib as L  # noqa: E402
from paper_2507_16784_b200.paging import stream_handle  # noqa: E402
from paper_2507_16784_b200.stepdesc import StepDesc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--max-mixed", type=int, default=40)
    a = ap.parse_args()
    eng, cfg, model = bench.build_engine(0, 64, 2)
    rt = eng.runtime
    rt.precapture()
    rt.recording = []
    while not eng.all_terminal():
        eng.step()
    records, rt.recording = rt.recording, None
    timed = set(bench.sampled_steps(len(records), a.steps, 5))
    mixed = [i for i in sorted(timed) if records[i][0].ext][: a.max_mixed]
    resident = rt.replay_upload(records)
    base = (StepDesc.EXT_US_PER_ITEM, StepDesc.EXT_US_PER_QBLOCK_BLOCK, StepDesc.DEC_US_PER_TOKEN)
    cands = [base, (3.0, 1.2, 4096 / 40e3)] + list(itertools.product((2.0, 4.0, 6.0, 8.0), (0.6, 0.7, 0.8, 0.9), (4096 / 32e3, 4096 / 36e3, 4096 / 40e3)))
    res = {c: [] for c in cands}
    st = stream_handle()
    D, hq, hkv = cfg.head_dim, cfg.heads, cfg.n_kv
    kl = model.pool_layer(rt.pool.K_layers, 0)
    vl = model.pool_layer(rt.pool.V_layers, 0)
    todo = set(mixed)
    for i, (sd, step, fw) in enumerate(resident):
        rt._execute(sd, step, fw)
        if i not in todo:
            continue
        torch.cuda.synchronize()
        for c in cands:
            StepDesc.EXT_US_PER_ITEM, StepDesc.EXT_US_PER_QBLOCK_BLOCK, StepDesc.DEC_US_PER_TOKEN = c
            ts = []
            for _ in range(3):
                rt.serial = (rt.serial % 0x7FFFFFFF) + 1
                sd.serial = rt.serial
                arr = sd.pack()
                dev = torch.from_numpy(arr).to(rt.dev)
                L.call("tim_attn_plan", dev.data_ptr(), rt.tables.data_ptr(), rt.tables.shape[1], rt.n_ctas,
                       rt.max_dec, D, rt.ws.data_ptr(), st)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                L.call("tim_attn_decode", dev.data_ptr(), 2, rt.q.data_ptr(), rt.ctx.data_ptr(), kl, vl,
                       rt.tables.data_ptr(), rt.tables.shape[1], hq, hkv, D, model.scale, rt.ws.data_ptr(),
                       rt.counters.data_ptr(), rt.n_ctas, rt.max_dec, cfg.tim_dtype, st)
                e1.record()
                ts.append((e0, e1))
            torch.cuda.synchronize()
            res[c].append(min(x.elapsed_time(y) for x, y in ts) * 1e3)
    out = sorted(((float(np.mean(v)), c) for c, v in res.items() if v))
    print(f"{len(mixed)} mixed steps; current {base}: {np.mean(res[base]):.1f} us")
    for us, c in out[:10]:
        print(f"  item {c[0]:.1f} us, block {c[1]:.2f} us, decode {4096 / c[2] / 1e3:.0f} KB/us per SM: {us:.1f} us")


if __name__ == "__main__":
    main()
