timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -3
timeout 120 python tools/attn_mixed_bench.py
timeout 120 python tools/attn_mixed_bench.py --ext 12 --n 180
timeout 120 python tools/attn_mixed_bench.py --ext 3 --n 60
timeout 120 python tools/attn_mixed_bench.py --ext 1 --n 20
