# full GPU suite + dense sweep + modes + launch lists (K3e rounds, u32 chunk starts)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
SZ_DENSE_RATES=0.0016,0.008,0.016,0.024,0.04,0.0789 timeout 900 python scripts/bench_dense.py > gpurun_out/dense.jsonl 2> gpurun_out/dense.err
timeout 900 python scripts/bench_modes.py > gpurun_out/modes.jsonl 2> gpurun_out/modes.err
for f in bf16 e5m2; do
  SZ_DEC_MARKED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dense_${f}.csv python scripts/profile_kernels.py $f $((1<<28)) 2 3 > /dev/null 2>&1
done
timeout 600 python scripts/bench_handoff.py --loopback --reps 3 > gpurun_out/handoff_loopback.json 2> gpurun_out/handoff.err
cat gpurun_out/pytest_gpu.log gpurun_out/dense.jsonl gpurun_out/modes.jsonl gpurun_out/handoff_loopback.json
for f in gpurun_out/launch_dense_*.csv; do echo $f; python scripts/launch_summary.py $f; done
tail -n 5 gpurun_out/dense.err gpurun_out/handoff.err
