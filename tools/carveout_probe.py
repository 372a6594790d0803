"""Does the shared-memory configuration left by the PRECEDING kernel change the
CUDA-event-bracketed time of a 148 x 320, ~200 KB-smem launch (the attention
kernel's shape)?  A = a small kernel launched just before the bracket (with 0
or 200 KB of dynamic smem, i.e. a small or a large carveout), B = the empty
attention-shaped grid between the events."""
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2507_16784_b200 import _lib as L  # noqa: E402

st = torch.cuda.current_stream().cuda_stream


def probe(a_smem, a_ctas=148, b_smem=203000, n=80):
    out = []
    torch.cuda._sleep(2_000_000)
    for _ in range(n):
        L.call("tim_noop", a_ctas, 256, a_smem, st)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        L.call("tim_noop", 148, 320, b_smem, st)
        b.record()
        out.append((a, b))
    torch.cuda.synchronize()
    v = sorted(x.elapsed_time(y) * 1000 for x, y in out[10:])
    return round(v[len(v) // 2], 2), round(v[0], 2)


for a_smem in (0, 48000, 100000, 203000):
    print(f"preceding smem {a_smem:6d}: bracketed empty attention-shaped grid median/min us", probe(a_smem))
print("b smem 0 after a smem 0:", probe(0, b_smem=0))
