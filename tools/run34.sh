timeout 600 ncu --set full --import-source on -k regex:attn_tiles -s 3 -c 1 -o gpurun_out/attn_mode2 python tools/attn_mixed_bench.py --layers 2 --only mode2 > /dev/null 2>&1
