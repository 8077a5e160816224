# A/B: K2b word copies + pack rewrite (base) vs previous commit (old), realistic + dense E5M2/BF16
set -x
rm -f gpurun_out/ab.txt
VARIANTS="base old" CONFIGS='"e5m2 top16 explicit c1024" "bf16 top16 explicit c1024" "e5m2 top8 3-bit c1024"' bash scripts/ab_variants.sh
