P="ncu --profile-from-start off --clock-control none"
TIMRUN_SKINNY=1 timeout 900 $P --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r1c_launches_decode_step_skinny.csv python tools/profile_step.py --rows 64 2>&1 | tail -1
for S in none gemm; do
  TIMRUN_SKINNY=1 TIMRUN_DIAG_SKIP=$S timeout 600 python bench.py --cpu-budget 0 --steps 200 > gpurun_out/ablsk_$S.json 2>/dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ablsk_$S.json')); print('skinny $S', round(d['ms_per_step'],3))"
done
