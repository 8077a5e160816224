# K6: one thread per 32 values, direct word stores (base) vs 8 values per
# thread through shared memory (k6old); parity first, then A/B and a launch list
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
VARIANTS="base k6old" CONFIGS='"e5m2 top8 3-bit c1024" "e5m2 top16 explicit c1024" "e4m3 top8 3-bit c1024"' bash scripts/ab_variants.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/k6_e5m2.csv python scripts/profile_kernels.py e5m2 $((1<<28)) 2 3 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/k6_e5m2.csv
