timeout 600 ncu --set full --import-source on -k regex:attn_ext_tc -s 2 -c 1 -o gpurun_out/attn_ext_tc python tools/attn_mixed_bench.py --layers 2 --only mode1 > /dev/null 2>&1
