timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -3
timeout 120 python tools/gemm_custom_bench.py
timeout 120 python tools/gemm_res_probe.py
