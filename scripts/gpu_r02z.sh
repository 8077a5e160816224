# A/B: 12-bit code-group table in the K3e decoder (t12) vs product (both with the cheaper non-dummy tracking)
set -x
rm -f gpurun_out/ab.txt
SZ_LIB_VARIANT=t12 timeout 900 python -m pytest tests/test_gpu_dense_escapes.py -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_robustness.py -x -q -k "k3e or dense" 2>&1 | tail -2
VARIANTS="base t12" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c1024"' bash scripts/ab_variants.sh
