timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 120 python tools/attn_microbench.py --live 724 --isolated
timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench53.json 2> gpurun_out/bench53.err; tail -1 gpurun_out/bench53.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench53.json")); r = d["roofline"]
print(d["value"], d["e2e"]["value"], d["ms_per_step"], r["frac"], r["event_floor_us"], r["achieved_net_of_event_floor"], r["decode_only_steps"]["ms_per_launch"])
PY
