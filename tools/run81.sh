timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench81.json 2>/dev/null
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench81.json")); r = d["roofline"]
print(round(d["value"]), round(d["e2e"]["value"]), d["ms_per_step"], r["frac"], r["decode_only_steps"]["ms_per_launch"], r["mixed_steps"]["ms_per_launch"], r["event_floor_us"])
PY
