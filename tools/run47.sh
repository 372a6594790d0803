timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_gemm_gpu.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench47a.json 2> gpurun_out/bench47a.err; tail -1 gpurun_out/bench47a.err
TIMRUN_SKINNY=1 timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench47b.json 2> gpurun_out/bench47b.err; tail -1 gpurun_out/bench47b.err
python - <<'PY'
import json
for f in ("gpurun_out/bench47a.json", "gpurun_out/bench47b.json"):
    d = json.load(open(f)); r = d["roofline"]
    print(f, d["value"], d["e2e"]["value"], d["ms_per_step"], r["frac"], r["event_floor_us"], r["achieved_net_of_event_floor"], r["decode_only_steps"]["ms_per_launch"])
PY
