#!/usr/bin/env bash
# Round-2 evidence run (one GPU): sanitizers at small shapes, the launch list of
# bench.py's value window (for roofline.traffic), full ncu captures of a
# decode-only and a mixed attention launch.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=tests/test_kernels_gpu.py
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -q -x -p no:cacheprovider \
  "$T::test_extend_tiles_bf16_matches_oracle[32-8-5-True-mixed]" "$T::test_decode_bf16_matches_oracle[32-8-3-True]" \
  "$T::test_page_ops_match_lifo_oracle" "$T::test_prune_compact_matches_apply" > gpurun_out/r2_synccheck.log 2>&1
echo "synccheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/r2_synccheck.log | tr '\n' ' ')"
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python -m pytest -q -x \
  -p no:cacheprovider "$T::test_decode_bf16_matches_oracle[16-4-3-False]" "$T::test_page_ops_match_lifo_oracle" \
  "$T::test_prune_compact_matches_apply" > gpurun_out/r2_racecheck.log 2>&1
echo "racecheck rc=$? $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY|passed|failed' gpurun_out/r2_racecheck.log | tr '\n' ' ')"
TIMRUN_PROFILE_TIMED=1 timeout 1500 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file gpurun_out/r2_launches_bench_timed.csv python bench.py --steps 12 --warmup 3 --cpu-budget 0 \
  > gpurun_out/r2_ncu_bench.log 2>&1
echo "launch list rc=$? lines $(wc -l < gpurun_out/r2_launches_bench_timed.csv)"
python tools/attention_traffic.py gpurun_out/r2_launches_bench_timed.csv "round 2" | tail -20
python tools/launch_summary.py gpurun_out/r2_launches_bench_timed.csv | head -14
P="ncu --profile-from-start off --clock-control none"
timeout 900 $P --set full --import-source on -k regex:"attn_(tiles|step)" -c 1 -o gpurun_out/r2_ncu_attn_decode_step python tools/profile_step.py --rows 64 > /dev/null 2>&1
timeout 900 $P --set full --import-source on -k regex:"attn_(tiles|step)" -c 1 -o gpurun_out/r2_ncu_attn_mixed_step python tools/profile_step.py --min-rows 600 > /dev/null 2>&1
ls -la gpurun_out/r2_ncu_attn_*
