python tools/rowkernel_bench.py
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench62.json 2> gpurun_out/bench62.err; tail -1 gpurun_out/bench62.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench62.json")); r = d["roofline"]
print(d["value"], d["e2e"]["value"], d["ms_per_step"], r["frac"], r["event_floor_us"], r["decode_only_steps"]["ms_per_launch"])
PY
