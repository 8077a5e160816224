# launch lists (per-kernel device time) for the slow ablation modes
set -x
for M in "bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c256"; do
  T=$(echo $M | tr ' ' '_')
  SZ_MODES_N=$((1<<28)) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/modes_$T.csv python scripts/bench_modes.py "$M" > gpurun_out/modes_$T.log 2>&1
done
timeout 900 python scripts/bench_modes.py "bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c256" "e4m3 top8 3-bit c1024"
