#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over the K1 (decode tiles +
# K6 merge), K2 (tcgen05 items, mode 1 and the mode-2 one-launch), K3 (RoPE +
# page store), K4 (prune compaction) and K5 (page ops) kernel tests at small
# shapes.  Logs go to gpurun_out/sanitize_<tool>.log; summaries are copied to
# profiles/ by hand.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=tests/test_kernels_gpu.py
SEL=(
  "$T::test_decode_bf16_matches_oracle[32-8-3-True]"
  "$T::test_decode_bf16_matches_oracle[32-8-1-False]"
  "$T::test_decode_bf16_matches_oracle[16-4-3-False]"
  "$T::test_extend_tiles_bf16_matches_oracle[32-8-5-False-mixed]"
  "$T::test_extend_tiles_bf16_matches_oracle[32-8-5-True-mixed]"
  "$T::test_rope_kv_store_matches_oracle[dtype1]"
  "$T::test_page_ops_match_lifo_oracle"
  "$T::test_prune_compact_matches_apply"
)
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  timeout "${SAN_TIMEOUT:-900}" compute-sanitizer --tool "$tool" $extra --print-limit 50 \
    --target-processes all python -m pytest -q -x -p no:cacheprovider "${SEL[@]}" \
    > "gpurun_out/sanitize_${tool}.log" 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitize_${tool}.log | tr '\n' ' ')"
done
