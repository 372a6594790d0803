# Diagnostics: K1 with the producer's copies removed (stale shared memory), so
# the consumer warps' own throughput shows; then the normal build.
TIMRUN_NVCC_FLAGS="-DTIM_CONSUMER_ONLY" python -c "from paper_2507_16784_b200.build import build; build(force=True)"
for C in 148 76; do timeout 120 python tools/attn_microbench.py --live 724 --ctas $C; done
python -c "from paper_2507_16784_b200.build import build; build(force=True)"
for C in 148 76; do timeout 120 python tools/attn_microbench.py --live 724 --ctas $C; done
timeout 120 python tools/attn_microbench.py --live 724 --isolated
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -1
