for S in none rope silu; do
  TIMRUN_DIAG_SKIP=$S timeout 600 python bench.py --cpu-budget 0 --steps 200 > gpurun_out/abl4_$S.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/abl4_$S.json')); print('$S', round(d['ms_per_step'],3))"
done
