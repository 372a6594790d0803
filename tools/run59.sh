P="ncu --profile-from-start off --clock-control none --cache-control none"
timeout 900 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/warm_decode.csv python tools/profile_step.py --rows 64 2>&1 | tail -1
timeout 900 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/warm_mixed.csv python tools/profile_step.py --min-rows 600 2>&1 | tail -1
