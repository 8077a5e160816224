# K2b sparse groups: TU tiles per warp step with every load in flight
# (base 16, tu8, tu4 = previous)
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense_escapes.py -x -q 2>&1 | tail -2
VARIANTS="base tu8 tu4" CONFIGS='"bf16 top16 explicit c1024" "e5m2 top16 explicit c1024" "bf16 top16 abs32" "bf16 top16 explicit c256"' bash scripts/ab_variants.sh
for v in base tu4; do
  if [ $v = base ]; then unset SZ_LIB_VARIANT; else export SZ_LIB_VARIANT=$v; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/k2b_$v.csv python scripts/profile_kernels.py bf16 $((1<<31)) 2 4 > /dev/null 2>&1
  python scripts/launch_summary.py gpurun_out/k2b_$v.csv | grep -E "gather|encode"
done
