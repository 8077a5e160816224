# K3e rounds: ping-pong batches / unconditional OR / uniform search branch
set -x
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_parity.py tests/test_gpu_robustness.py -x -q -k "k3e or dense" 2>&1 | tail -2 > gpurun_out/pytest_u.log
for f in bf16 e5m2; do
  SZ_DEC_MARKED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dense_${f}.csv python scripts/profile_kernels.py $f $((1<<28)) 2 3 > /dev/null 2>&1
done
SZ_DENSE_PATHS=1 SZ_DENSE_RATES=0.0789 timeout 900 python scripts/bench_dense.py > gpurun_out/dense_u.jsonl 2> gpurun_out/dense.err
cat gpurun_out/pytest_u.log gpurun_out/dense_u.jsonl
for f in gpurun_out/launch_dense_*.csv; do echo $f; python scripts/launch_summary.py $f | grep -E "decode|marks"; done
