timeout 120 python tools/attn_mixed_bench.py
timeout 120 python tools/attn_mixed_bench.py --ext 12 --n 180
timeout 120 python tools/attn_mixed_bench.py --ext 3 --n 60
timeout 120 python tools/attn_mixed_bench.py --ext 0
