# A/B: XOR-swizzled 12-bit code-group table (x12) vs plain (base)
set -x
rm -f gpurun_out/ab.txt
SZ_LIB_VARIANT=x12 timeout 900 python -m pytest tests/test_gpu_dense_escapes.py -x -q 2>&1 | tail -2
VARIANTS="base x12" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024"' bash scripts/ab_variants.sh
