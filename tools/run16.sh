timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
python tools/attn_microbench.py --live 724
python tools/attn_microbench.py --live 309
TIMRUN_PHASES=1 timeout 900 python bench.py --steps 100 --warmup 3 --skip 600 --cpu-budget 0 2>&1 | tail -30
