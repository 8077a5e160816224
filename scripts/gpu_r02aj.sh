# A/B: 8 rounds in flight in K3e and K2b's dense word copy (u8) vs 4 (base)
set -x
rm -f gpurun_out/ab.txt
SZ_LIB_VARIANT=u8 timeout 900 python -m pytest tests/test_gpu_dense_escapes.py -x -q 2>&1 | tail -1
VARIANTS="base u8" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024"' bash scripts/ab_variants.sh
