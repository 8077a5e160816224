# launch lists of the codec at chunk 1024 vs 65536 (2^28 BF16 words)
for c in 1024 65536; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_chunk$c.csv python scripts/profile_kernels.py bf16 $((1<<28)) 3 4 $c > /dev/null 2>&1
  python scripts/launch_summary.py gpurun_out/launches_chunk$c.csv | head -8
done
