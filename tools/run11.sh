python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
python tools/attn_microbench.py --live 724 --trace
python tools/attn_microbench.py --live 309 --trace
python tools/attn_microbench.py --live 2000
python tools/attn_microbench.py --live 724 --batch 1 --trace
python -m pytest tests/test_engine_gpu.py -x -q 2>&1 | tail -2
TIMRUN_PHASES=1 timeout 900 python bench.py --steps 60 --warmup 3 --skip 600 --cpu-budget 0 2>&1 | tail -36
