#!/usr/bin/env bash
# The GPU session used for this round's evidence (run through gpurun from the
# repo root): parity suite, smoke, bench line, ncu launch lists and full
# captures of the attention launches of a decode-only and a mixed step.
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/gpu_checks.sh'
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
P="ncu --profile-from-start off --clock-control none"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv"
timeout 900 $P $M --log-file gpurun_out/launches_decode_step.csv python tools/profile_step.py --rows 64
timeout 900 $P $M --log-file gpurun_out/launches_mixed_step.csv python tools/profile_step.py --min-rows 600
timeout 900 $P --set full --import-source on -k regex:"attn_(tiles|step)" -c 1 -o gpurun_out/ncu_attn_decode_step python tools/profile_step.py --rows 64
timeout 900 $P --set full --import-source on -k regex:"attn_(tiles|step)" -c 1 -o gpurun_out/ncu_attn_mixed_step python tools/profile_step.py --min-rows 600
timeout 600 python tools/bench_configs.py --config c5 --skip 1500 --steps 100 > gpurun_out/c5.json
timeout 1500 python tools/bench_configs.py --config c4 --skip 600 --steps 100 > gpurun_out/c4.json
