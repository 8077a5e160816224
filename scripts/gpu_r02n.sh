# A/B: FP8 K2a with 7 writer warps (7 scan slots) vs the product build
set -x
rm -f gpurun_out/ab.txt
VARIANTS="base w7" CONFIGS='"e5m2 top8 3-bit c1024" "e5m2 top16 explicit c1024" "e4m3 top8 3-bit c1024"' bash scripts/ab_variants.sh
