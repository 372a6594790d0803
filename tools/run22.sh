timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -3
timeout 120 python tools/gemm_custom_bench.py
timeout 300 ncu --set full --import-source on -k regex:gemm_skinny -s 20 -c 1 -o gpurun_out/gemm_tc python tools/gemm_custom_bench.py > /dev/null 2>&1
ls gpurun_out
