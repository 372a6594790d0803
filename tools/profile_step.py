"""Profile steady-state C2 engine steps under ncu (run with
`ncu --profile-from-start off ...`): after --skip steps (same default as
bench.py), the profiler window opens around the next step whose batched
forward has exactly --rows rows (64 = a decode-only step; 0 = any step)."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip", type=int, default=1500)
    ap.add_argument("--rows", type=int, default=64)
    ap.add_argument("--min-rows", type=int, default=0, help="profile the next step with >= this many rows")
    a = ap.parse_args()
    eng, cfg, model = bench.build_engine(0, 64, 2)
    rt = eng.runtime
    rt.precapture()
    for _ in range(a.skip):
        eng.step()
    torch.cuda.synchronize()
    orig = rt.run_step
    state = {"done": False, "rows": None}

    def run_step(sd, forward=True):
        want = (a.min_rows and sd.n_rows >= a.min_rows) or (not a.min_rows and (a.rows == 0 or sd.n_rows == a.rows))
        if state["done"] or not forward or not want:
            return orig(sd, forward)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        out = orig(sd, forward)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        state["done"], state["rows"] = True, sd.n_rows
        return out

    rt.run_step = run_step
    while not state["done"]:
        eng.step()
    print(f"profiled one step with {state['rows']} rows", file=sys.stderr)


if __name__ == "__main__":
    main()
