timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -1
for P in "" "--no-plan"; do timeout 120 python tools/attn_microbench.py --live 724 $P; timeout 120 python tools/attn_microbench.py --live 724 --isolated $P; timeout 120 python tools/attn_microbench.py --live 724 --trace $P 2>&1 | head -1; done
