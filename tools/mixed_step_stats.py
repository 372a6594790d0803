"""Composition of bench.py's timed mixed steps (C2): decode tiles / tokens, K2
items, their 64-key blocks x q-blocks, and the mode-2 split the cost model
picks.  usage: python tools/mixed_step_stats.py"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    eng, cfg, model = bench.build_engine(0, 64, 2)
    rt = eng.runtime
    rt.recording = []
    while not eng.all_terminal():
        eng.step()
    records, rt.recording = rt.recording, None
    timed = bench.sampled_steps(len(records), 200, 5)
    rows = []
    for i in timed:
        sd = records[i][0]
        if not sd.ext:
            continue
        sd.pack()
        dec_tok = sum(d[2] for d in sd.dec)
        blocks = sum(((e[2] + 63) // 64) * ((e[3] + 31) // 32) for e in sd.ext)
        segs = [(sg[1], sg[2]) for sg in sd.segs if sg[2] > 1]
        rows.append((len(sd.dec), dec_tok, len(sd.ext), blocks, sd.offsets["split_dec_ctas"],
                     sd.offsets["split_ext_ctas"], segs))
    a = np.array([r[:6] for r in rows], dtype=float)
    print(f"{len(rows)} mixed steps of {len(timed)} timed")
    print("mean: dec tiles %.0f, dec tokens %.0f, items %.0f, item-blocks %.0f, split dec/ext %.0f/%.0f" %
          tuple(a.mean(axis=0)))
    for q in (10, 50, 90):
        print(f"p{q}: items {np.percentile(a[:, 2], q):.0f}, item-blocks {np.percentile(a[:, 3], q):.0f}, "
              f"ext CTAs {np.percentile(a[:, 5], q):.0f}")
    for r in rows[:12]:
        print(r[:6], "multi-token segments (m, n):", r[6][:6])


if __name__ == "__main__":
    main()
