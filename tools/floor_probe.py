import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2507_16784_b200 import _lib as L
torch.cuda.init()
st = torch.cuda.current_stream().cuda_stream
def probe(smem, threads=288, sleep=True, n=60):
    out = []
    if sleep: torch.cuda._sleep(4_000_000)
    for i in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); L.call("tim_noop", 148, threads, smem, st); b.record(); out.append((a, b))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) for a, b in out[10:])
    return round(v[len(v)//2] * 1000, 2), round(v[0] * 1000, 2)
for smem in (0, 100000, 203000, 230000):
    print(smem, "sleep", probe(smem), "nosleep", probe(smem, sleep=False))
# two back-to-back noops inside one bracket
out=[]
torch.cuda._sleep(4_000_000)
for i in range(60):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); L.call("tim_noop", 148, 288, 203000, st); L.call("tim_noop", 148, 288, 203000, st); b.record(); out.append((a,b))
torch.cuda.synchronize()
v = sorted(a.elapsed_time(b) for a, b in out[10:]); print("two noops", v[len(v)//2]*1000)
