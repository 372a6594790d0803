timeout 600 ncu --set full --import-source on -k regex:attn_tiles -s 20 -c 1 -o gpurun_out/attn_mixed python tools/attn_mixed_bench.py --layers 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:attn_tiles -s 20 -c 1 -o gpurun_out/attn_dec python tools/attn_microbench.py --layers 2 --iters 12 > /dev/null 2>&1
ls -la gpurun_out
