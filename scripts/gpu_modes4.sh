set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; tail -3 gpurun_out/pt_all.log
timeout 900 python scripts/bench_modes.py "bf16 top16 explicit c1024" "bf16 top15 sentinel c1024" "bf16 top16 abs32" "e5m2 top16 explicit c1024" > gpurun_out/modes_sub.jsonl 2>&1; cat gpurun_out/modes_sub.jsonl
for M in sentinel abs32; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/modes_$M.csv python scripts/profile_kernels.py bf16 $((1<<28)) 2 4 1024 $M > gpurun_out/pm_$M.log 2>&1
done
