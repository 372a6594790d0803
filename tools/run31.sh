timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -2
timeout 120 python tools/gemm_custom_bench.py
TIMRUN_SKINNY=1 timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench31.json 2> gpurun_out/bench31.err; tail -3 gpurun_out/bench31.err; cat gpurun_out/bench31.json
