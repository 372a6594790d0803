timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -5
for L in 309 724 2000; do timeout 120 python tools/attn_microbench.py --live $L --trace; done
timeout 120 python tools/attn_microbench.py --live 724 --batch 512 --trace
timeout 120 python tools/attn_microbench.py --live 724 --trace --dump > gpurun_out/dump28.txt
