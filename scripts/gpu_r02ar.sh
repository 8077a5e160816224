# K4 decode warps: wait for the stagers after the first slot's unpack (base)
# vs before it (eager)
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
VARIANTS="base eager" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c1024" "e5m2 top16 explicit c1024" "bf16 top15 sentinel c1024" "bf16 top16 abs32"' bash scripts/ab_variants.sh
