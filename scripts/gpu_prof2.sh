set -x
python scripts/profile_e2e.py $((1<<31)) e5m2 > gpurun_out/e2e_phases_e5m2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'encode_tiles|decode_persistent' -s 2 -c 2 -o gpurun_out/prof_r01f_e5m2 python scripts/profile_kernels.py e5m2 $((1<<28)) 2 > gpurun_out/prof_e5m2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'encode_tiles|decode_persistent' -s 2 -c 2 -o gpurun_out/prof_r01f_bf16 python scripts/profile_kernels.py bf16 $((1<<28)) 2 > gpurun_out/prof_bf16.log 2>&1
cat gpurun_out/e2e_phases_e5m2.txt
