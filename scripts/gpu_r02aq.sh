# K2a dense warps: warp-aggregated escape-record reservation (base) vs one
# shared atomic per lane with escapes (escatom)
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
VARIANTS="base escatom" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c1024" "e5m2 top16 explicit c1024"' bash scripts/ab_variants.sh
