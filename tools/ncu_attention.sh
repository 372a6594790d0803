P="ncu --profile-from-start off --clock-control none"
timeout 900 $P --set full --import-source on -k regex:"attn_(tiles|step)" -c 1 -o gpurun_out/ncu_attn_decode_step python tools/profile_step.py --rows 64
timeout 900 $P --set full --import-source on -k regex:"attn_(tiles|step)" -c 1 -o gpurun_out/ncu_attn_mixed_step python tools/profile_step.py --min-rows 600
