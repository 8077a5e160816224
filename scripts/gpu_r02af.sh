# A/B: pack grid 296 (p296) vs capacity-sized (base) vs previous commit (old), E5M2 realistic encode
set -x
rm -f gpurun_out/ab.txt
VARIANTS="base p296 old" CONFIGS='"e5m2 top16 explicit c1024" "e5m2 top8 3-bit c1024"' bash scripts/ab_variants.sh
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_e5real.csv python scripts/profile_kernels.py e5m2 $((1<<28)) 2 4 > /dev/null 2>&1
SZ_LIB_VARIANT=old timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_e5real_old.csv python scripts/profile_kernels.py e5m2 $((1<<28)) 2 4 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launch_e5real.csv; python scripts/launch_summary.py gpurun_out/launch_e5real_old.csv
