# source-level captures: E5M2 top-8 3-bit encode (K2a) and decode (K4, K3e
# path) after the stager change
set -x
timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'encode_tiles|decode_persistent' -s 4 -c 2 -o gpurun_out/e5dense_ap python scripts/profile_kernels.py e5m2 $((1<<28)) 3 3 > gpurun_out/ap_prof.log 2>&1
tail -3 gpurun_out/ap_prof.log
ls -la gpurun_out | tail -3
