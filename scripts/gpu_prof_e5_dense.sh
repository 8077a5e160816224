timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'encode_tiles' -s 1 -c 1 \
  -o gpurun_out/prof_e5dense python scripts/profile_kernels.py e5m2 $((1<<28)) 2 3 > gpurun_out/prof_e5dense.log 2>&1
tail -2 gpurun_out/prof_e5dense.log
