set -x
python tools/attn_microbench.py --live 724
python tools/attn_microbench.py --live 309
python tools/attn_microbench.py --live 2000
python tools/attn_microbench.py --live 724 --batch 512
ncu --set full --clock-control none --import-source on -k regex:attn_decode -s 8 -c 1 -o gpurun_out/prof_decode_r1 python tools/attn_microbench.py --live 724 --iters 2 > gpurun_out/ncu_decode.log 2>&1
tail -3 gpurun_out/ncu_decode.log
python -m pytest tests/ -x -q -m gpu 2>&1 | tail -5
timeout 900 python bench.py --steps 60 --warmup 3 --skip 600 --cpu-budget 0 2>&1 | tail -3
TIMRUN_GRAPHS=0 timeout 900 python bench.py --steps 60 --warmup 3 --skip 600 --cpu-budget 0 2>&1 | tail -3
