"""Profile the engine's host-side step planning on CPU (device calls stubbed).

Runs the C2 workload (64 tool_chain_tree(32) requests, T=2) through
Engine.step() with a fake pool/runtime that only packs the step descriptor,
and prints the per-step host cost and the cProfile top entries.
"""

import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2507_16784_b200 as tr  # noqa: E402
from paper_2507_16784_b200 import paging  # noqa: E402
from paper_2507_16784_b200.traces import load_corpus, make_trace_from_text  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]


class FakePool(paging.DevicePagePool):
    def __init__(self, capacity):  # no device state
        self.capacity = capacity
        self._sp = capacity
        self._codes, self._owners = {}, []


class FakeRuntime:
    def __init__(self):
        self.launches = 0

    def run_step(self, sd, forward=True):
        sd.pack()
        return None


class FakeBackend:
    position_limit = 40960
    has_weights = False

    def make_pool(self, capacity):
        return FakePool(capacity)

    def runtime(self, pool, max_slots, logical_cap):
        return FakeRuntime()

    def plan_attention(self, sd, slot, m, n, row_off):
        sd.segs.append((slot, m, n, row_off))
        for q0 in range(0, n, 4):
            nq = min(4, n - q0)
            sd.dec.append((row_off + q0, slot, m + q0 + nq, nq, m, 0))


def main(steps=800):
    docs = load_corpus(ROOT / "tests" / "golden" / "corpus_tool_chain32.json.gz")[:64]
    eng = tr.Engine(FakeBackend(), tr.BatchConfig(max_batch=64, buffer_threshold=2,
                                                  position_limit=40960, pool_pages=64 * 1600,
                                                  check_masks=False, max_output_tokens=20000))
    for i, d in enumerate(docs):
        t = make_trace_from_text(d)
        eng.submit(f"q0.{i}:", [tr.ToolSpec(n) for n in t.tool_names], script=t.script,
                   tool_responses=t.tool_responses)
    prof = cProfile.Profile()
    t0 = time.perf_counter()
    prof.enable()
    for _ in range(steps):
        eng.step()
    prof.disable()
    dt = time.perf_counter() - t0
    print(f"{steps} steps, {dt * 1000 / steps:.3f} ms/step host planning (under cProfile)")
    pstats.Stats(prof).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 800)
