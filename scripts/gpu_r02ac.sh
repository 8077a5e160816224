# K2b dense path as warp word copies: tests + modes + launch lists
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 900 python scripts/bench_modes.py > gpurun_out/modes.jsonl 2> gpurun_out/modes.err
for f in bf16 e5m2; do
  SZ_DEC_MARKED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dense_${f}.csv python scripts/profile_kernels.py $f $((1<<28)) 2 3 > /dev/null 2>&1
done
cat gpurun_out/pytest_gpu.log gpurun_out/modes.jsonl
for f in gpurun_out/launch_dense_*.csv; do echo $f; python scripts/launch_summary.py $f | grep -E "gather|encode|pack"; done
