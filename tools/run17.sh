timeout 900 python bench.py --steps 100 --warmup 3 --skip 600 --cpu-budget 0 2>&1 | grep -v "^{" | tail -5
timeout 1200 python tools/bench_configs.py --config c5 --skip 600 --steps 100 2>&1 | tail -2
timeout 600 python tools/bench_configs.py --config c1 2>&1 | tail -2
timeout 1200 python tools/bench_configs.py --config c4 --skip 2000 --steps 200 2>&1 | tail -2
