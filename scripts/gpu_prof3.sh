set -x
F=${F:-e5m2}
TAG=${TAG:-r01g}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'encode_tiles|decode_persistent' -s 2 -c 2 -o gpurun_out/prof_${TAG}_$F python scripts/profile_kernels.py $F $((1<<28)) 2 > gpurun_out/prof_$F.log 2>&1
