set -x
for M in sentinel abs32; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/modes_$M.csv python scripts/profile_kernels.py bf16 $((1<<28)) 2 4 1024 $M > gpurun_out/pm_$M.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'decode_persistent|marks' -s 2 -c 2 -o gpurun_out/prof_r01s_$M python scripts/profile_kernels.py bf16 $((1<<28)) 2 4 1024 $M > /dev/null 2>&1
done
