timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -2
for L in 309 724 2000; do timeout 120 python tools/attn_microbench.py --live $L; timeout 120 python tools/attn_microbench.py --live $L --isolated; done
timeout 120 python tools/attn_microbench.py --live 724 --trace --dump > gpurun_out/dump54.txt
timeout 120 python tools/attn_mixed_bench.py
