P="ncu --profile-from-start off --clock-control none"
timeout 900 $P --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r1c_launches_decode_step.csv python tools/profile_step.py --rows 64 2>&1 | tail -1
timeout 900 $P --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r1c_launches_mixed_step.csv python tools/profile_step.py --min-rows 600 2>&1 | tail -1
timeout 900 $P --set full --import-source on -k regex:attn_ -c 1 -o gpurun_out/r1c_attn_decode_step python tools/profile_step.py --rows 64 2>&1 | tail -1
timeout 900 $P --set full --import-source on -k regex:attn_ -c 1 -o gpurun_out/r1c_attn_mixed_step python tools/profile_step.py --min-rows 600 2>&1 | tail -1
