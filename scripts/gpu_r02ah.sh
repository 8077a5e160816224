# A/B: dense escape loop unrolled by 2 (base) vs previous commit (old)
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
VARIANTS="base old" CONFIGS='"e5m2 top16 explicit c1024" "e5m2 top8 3-bit c1024" "bf16 top8 3-bit c1024" "bf16 top16 explicit c1024"' bash scripts/ab_variants.sh
