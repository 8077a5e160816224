# Decoder stagers: values run with every load in flight (vs a loop of one
# latency per 32 words: stgold) and back-off idle waits (vs sleeping
# try_wait: stgspin); both old: stgboth.  Parity, then A/B.
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_robustness.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
VARIANTS="base stgold stgspin stgboth" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c1024" "e5m2 top16 explicit c1024" "bf16 top15 sentinel c1024"' bash scripts/ab_variants.sh
