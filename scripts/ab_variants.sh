# A/B of variant builds (python -c "from paper_2605_01708_b200 import _build;
# _build.build(variant=NAME, defines=(...))"): alternating bench_modes runs
# on one box.  usage: VARIANTS="base cap2048" CONFIGS="..." bash scripts/ab_variants.sh
set -x
VARIANTS=${VARIANTS:-"base"}
for round in 1 2; do
  for v in $VARIANTS; do
    if [ "$v" = base ]; then unset SZ_LIB_VARIANT; else export SZ_LIB_VARIANT=$v; fi
    eval timeout 600 python scripts/bench_modes.py $CONFIGS 2>/dev/null | sed "s/^/$v /" >> gpurun_out/ab.txt
  done
done
unset SZ_LIB_VARIANT
cat gpurun_out/ab.txt
