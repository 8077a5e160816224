# K2b escape-dense runs: 16-byte loads (base) vs 4-byte words (k2bword)
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
VARIANTS="base k2bword" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c1024" "e5m2 top16 explicit c1024"' bash scripts/ab_variants.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/k2b_e5m2.csv python scripts/profile_kernels.py e5m2 $((1<<28)) 2 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/k2b_e5m2.csv
