set -x
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:'escape_gather' -s 1 -c 1 -o gpurun_out/prof_r01w_gather python scripts/profile_kernels.py bf16 $((1<<31)) 2 > gpurun_out/prof_gather.log 2>&1
