timeout 1500 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py 2>&1 | tail -8
python tools/gemm_microbench.py default
python tools/gemm_microbench.py cublas
DISABLE_ADDMM_CUDA_LT=1 python tools/gemm_microbench.py default
