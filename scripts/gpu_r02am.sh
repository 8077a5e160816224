# K3e leaner rounds (register chunk starts, byte value table): parity, A/B
# against the previous rounds (k3eold), ncu of the K3e path's K4 + K3e
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_robustness.py -x -q 2>&1 | tail -2
VARIANTS="base k3eold" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024"' bash scripts/ab_variants.sh
SZ_DEC_MARKED=1 timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'decode_persistent|escape_marks' -s 2 -c 2 -o gpurun_out/k3e_am_e5m2 python scripts/profile_kernels.py e5m2 $((1<<28)) 2 3 > /dev/null 2>&1
ls -la gpurun_out | tail -5
