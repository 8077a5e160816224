# ncu --set full of the escape-heavy kernels: BF16 top-8 3-bit (eps 6.9%)
set -x
TAG=${TAG:-r01j}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'decode_persistent|escape_heavy|escape_gather' -s 3 -c 3 -o gpurun_out/prof_${TAG}_heavy python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > gpurun_out/prof_heavy.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'encode_tiles' -s 1 -c 1 -o gpurun_out/prof_${TAG}_c256 python scripts/profile_kernels.py bf16 $((1<<28)) 1 4 256 > gpurun_out/prof_c256.log 2>&1
