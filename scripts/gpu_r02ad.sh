# K2b dense word copies with 4 rounds in flight + coalesced pack_values
set -x
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_ad.log
timeout 600 python scripts/bench_modes.py "bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "e5m2 top16 explicit c1024" > gpurun_out/modes_ad.jsonl 2>/dev/null
for f in bf16 e5m2; do
  SZ_DEC_MARKED=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dense_${f}.csv python scripts/profile_kernels.py $f $((1<<28)) 2 3 > /dev/null 2>&1
done
cat gpurun_out/pytest_ad.log gpurun_out/modes_ad.jsonl
for f in gpurun_out/launch_dense_bf16.csv gpurun_out/launch_dense_e5m2.csv; do echo $f; python scripts/launch_summary.py $f | grep -E "gather|encode|pack"; done
