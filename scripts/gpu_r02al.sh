# A/B: K3e instantiation at 2 CTAs x 5 stages (k2c) vs 3 CTAs x 3-4 stages (base)
set -x
rm -f gpurun_out/ab.txt
SZ_LIB_VARIANT=k2c timeout 900 python -m pytest tests/test_gpu_dense_escapes.py -x -q 2>&1 | tail -1
VARIANTS="base k2c" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024"' bash scripts/ab_variants.sh
