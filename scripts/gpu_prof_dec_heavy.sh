set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'decode_persistent' -s 1 -c 1 -o gpurun_out/prof_r01v_dec python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > gpurun_out/prof_heavy.log 2>&1
