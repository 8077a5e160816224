set -x
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:'offsets_kernel' -s 0 -c 4 -o gpurun_out/prof_r01v_scan python scripts/profile_kernels.py bf16 $((1<<31)) 3 > gpurun_out/prof_scan.log 2>&1
