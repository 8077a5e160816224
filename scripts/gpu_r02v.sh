# A/B: E5M2 decode at 3 CTAs/SM (56 regs, 3 stages) vs product
set -x
rm -f gpurun_out/ab.txt
VARIANTS="base e53" CONFIGS='"e5m2 top16 explicit c1024" "e5m2 top8 3-bit c1024"' bash scripts/ab_variants.sh
