for Q in 2 1; do
  sed -i "s/^constexpr int QBLK = [0-9];/constexpr int QBLK = $Q;/" paper_2507_16784_b200/csrc/attention_tc.cuh
  python -c "from paper_2507_16784_b200.build import build; build(force=True)" 2>&1 | grep -i error
  timeout 900 python bench.py --cpu-budget 0 > gpurun_out/bench69_$Q.json 2>/dev/null
  python - <<PY
import json
d = json.load(open("gpurun_out/bench69_$Q.json")); r = d["roofline"]
print("QBLK=$Q", round(d["value"]), r["frac"], r["decode_only_steps"]["ms_per_launch"], r["mixed_steps"]["ms_per_launch"], r["mixed_steps"]["bytes_per_launch"])
PY
done
