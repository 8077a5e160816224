# ncu --set full + source of the E5M2 encoder (K2a) and decoder (K4) at 2^29 words
set -x
timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'encode_tiles|decode_persistent' -s 2 -c 2 \
  -o gpurun_out/prof_e5 python scripts/profile_kernels.py e5m2 $((1<<29)) 3 > gpurun_out/prof_e5.log 2>&1
ls -la gpurun_out
