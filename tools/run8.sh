python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
python tools/attn_microbench.py --live 724
python tools/attn_microbench.py --live 309
python tools/attn_microbench.py --live 2000
python tools/attn_microbench.py --live 724 --batch 512
TIMRUN_PHASES=1 timeout 900 python bench.py --steps 60 --warmup 3 --skip 600 --cpu-budget 0 2>&1 | tail -16
