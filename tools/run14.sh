python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
python tools/attn_microbench.py --live 724 --trace
TIMRUN_PHASES=1 timeout 900 python bench.py --steps 100 --warmup 3 --skip 600 --cpu-budget 0 2>&1 | tail -30
