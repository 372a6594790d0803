for C in "2.0,0.8" "4.0,1.6" "6.0,2.8"; do
  TIMRUN_EXT_COST=$C timeout 900 python bench.py --cpu-budget 0 --steps 100 > gpurun_out/bench71.json 2>/dev/null
  python - <<PY
import json
d = json.load(open("gpurun_out/bench71.json")); r = d["roofline"]
print("cost $C", round(d["value"]), r["frac"], r["decode_only_steps"]["ms_per_launch"], r["mixed_steps"]["ms_per_launch"])
PY
done
