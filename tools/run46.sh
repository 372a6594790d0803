timeout 300 python tools/bench_configs.py --config c1 > gpurun_out/c1.json 2> gpurun_out/c1.err; tail -2 gpurun_out/c1.err; cat gpurun_out/c1.json
timeout 900 python tools/bench_configs.py --config c5 --skip 1500 --steps 100 > gpurun_out/c5.json 2> gpurun_out/c5.err; tail -2 gpurun_out/c5.err; cat gpurun_out/c5.json
timeout 1500 python tools/bench_configs.py --config c4 --skip 600 --steps 100 > gpurun_out/c4.json 2> gpurun_out/c4.err; tail -3 gpurun_out/c4.err; cat gpurun_out/c4.json
timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench46.json 2> gpurun_out/bench46.err; tail -2 gpurun_out/bench46.err; cat gpurun_out/bench46.json
