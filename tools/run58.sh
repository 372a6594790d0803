timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for S in none rope,silu; do
  TIMRUN_DIAG_SKIP=$S timeout 600 python bench.py --cpu-budget 0 --steps 200 > gpurun_out/abl3_$S.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/abl3_$S.json')); print('$S', round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], d['roofline']['decode_only_steps']['ms_per_launch'])"
done
