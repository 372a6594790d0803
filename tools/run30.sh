timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench30.json 2> gpurun_out/bench30.err; tail -4 gpurun_out/bench30.err; cat gpurun_out/bench30.json
