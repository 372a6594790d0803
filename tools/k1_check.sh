timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -1
timeout 120 python tools/attn_microbench.py --live 724
timeout 120 python tools/attn_microbench.py --live 724 --isolated
timeout 120 python tools/attn_microbench.py --live 724 --trace --dump > gpurun_out/dump88.txt
