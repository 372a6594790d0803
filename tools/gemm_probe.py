import torch, time
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = True
d = "cuda"
shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "up": (12288, 4096), "down": (4096, 12288)}
def bench(f, n=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1000
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=d)
for M in (64, 128):
    for name, (N, K) in shapes.items():
        ws = [torch.randn(N, K, device=d, dtype=torch.bfloat16) for _ in range(8)]  # > L2 in rotation
        x = torch.randn(M, K, device=d, dtype=torch.bfloat16)
        y = torch.empty(M, N, device=d, dtype=torch.bfloat16)
        i = [0]
        def f():
            i[0] = (i[0] + 1) % 8
            torch.matmul(x, ws[i[0]].t(), out=y)
        us = bench(f)
        print(f"M={M} {name:5s} N={N} K={K}: {us:6.1f} us  {N*K*2/us/1e3:7.0f} GB/s")
for name, (N, K) in shapes.items():
    ws = [torch.randn(N, K, device=d, dtype=torch.bfloat16) for _ in range(8)]
    x = torch.randn(64, K, device=d, dtype=torch.bfloat16)
    def g(): 
        for w in ws: torch.matmul(x, w.t())
    us = bench(g, 20) / 8
    print(f"back-to-back 8 different weights, M=64 {name}: {us:6.1f} us  {N*K*2/us/1e3:7.0f} GB/s")
