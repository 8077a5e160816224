set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'escape_gather|offsets_kernel' -s 2 -c 2 -o gpurun_out/prof_r01u_small python scripts/profile_kernels.py bf16 $((1<<31)) 2 > gpurun_out/prof_small.log 2>&1
