timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench36.json 2> gpurun_out/bench36.err; tail -3 gpurun_out/bench36.err; cat gpurun_out/bench36.json
