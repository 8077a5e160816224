# Decoder stagers, K3e values run staged at its global 16-byte alignment
# (aligned quad stores, decode warps read from vshift): parity, then A/B
# against the previous copy loop (stgold) and both previous (stgboth).
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
VARIANTS="base stgold stgboth" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c1024" "e5m2 top16 explicit c1024" "bf16 top15 sentinel c1024"' bash scripts/ab_variants.sh
