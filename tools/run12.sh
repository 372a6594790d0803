python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
python tools/attn_microbench.py --live 724 --trace
python tools/attn_microbench.py --live 309 --trace
timeout 900 python bench.py --steps 100 --warmup 3 --skip 600 --cpu-budget 10 2>&1 | tail -6
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/profile_step.py --skip 600 > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_decode -c 1 -o gpurun_out/prof_decode_step python tools/profile_step.py --skip 600 > gpurun_out/ncu_step.log 2>&1
tail -2 gpurun_out/ncu_step.log
