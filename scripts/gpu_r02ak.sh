# A/B: K3e with two ordinals per lane per round (base) vs one (old)
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_robustness.py tests/test_gpu_parity.py -x -q -k "k3e or dense" 2>&1 | tail -1
VARIANTS="base old" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024"' bash scripts/ab_variants.sh
SZ_DEC_MARKED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_k3e2.csv python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launch_k3e2.csv | grep -E "marks|decode"
