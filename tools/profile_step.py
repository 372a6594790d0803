"""Profile one steady-state C2 engine step under ncu (profiling window only
around the chosen step; run with `ncu --profile-from-start off ...`)."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip", type=int, default=600)
    ap.add_argument("--decode-only", action="store_true", help="profile the next step with 64 rows")
    a = ap.parse_args()
    eng, cfg, model = bench.build_engine(0, 64, 2)
    eng.runtime.precapture()
    for _ in range(a.skip):
        eng.step()
    # find a decode-only step: plan ahead without executing would change state; instead
    # step until the *planned* row count is 64 by peeking at the last step's rows
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    eng.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled one step", file=sys.stderr)


if __name__ == "__main__":
    main()
