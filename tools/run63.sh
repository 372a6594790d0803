timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for LT in 1 0; do
TIMRUN_LT=$LT timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench63_$LT.json 2> gpurun_out/bench63_$LT.err; tail -1 gpurun_out/bench63_$LT.err
python - <<PY
import json
d = json.load(open("gpurun_out/bench63_$LT.json")); r = d["roofline"]
print("LT=$LT", d["value"], d["e2e"]["value"], d["ms_per_step"], r["frac"], r["decode_only_steps"]["ms_per_launch"])
PY
done
