# group-wise escape merge in K4 + 32-bit K3e: tests, rate sweep, modes, launch lists
set -x
timeout 1500 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_paged.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_k3e.log
SZ_DENSE_RATES=0.0016,0.004,0.008,0.016,0.04,0.0789 timeout 900 python scripts/bench_dense.py > gpurun_out/dense.jsonl 2> gpurun_out/dense.err
timeout 600 python scripts/bench_modes.py "bf16 top16 explicit c1024" "bf16 top8 3-bit c1024" "bf16 top15 sentinel c1024" "e5m2 top16 explicit c1024" "e5m2 top8 3-bit c1024" "e4m3 top8 3-bit c1024" > gpurun_out/modes_j.jsonl 2> gpurun_out/modes_j.err
for path in 0 1; do
  SZ_DEC_MARKED=$path timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dense_p$path.csv python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > /dev/null 2>&1
  SZ_DEC_MARKED=$path timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dense_e5_p$path.csv python scripts/profile_kernels.py e5m2 $((1<<28)) 2 3 > /dev/null 2>&1
done
SZ_DEC_MARKED=1 timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'decode_persistent|escape_marks' -s 2 -c 2 -o gpurun_out/dense_k3e python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > gpurun_out/prof_dense.log 2>&1
cat gpurun_out/pytest_k3e.log gpurun_out/dense.jsonl gpurun_out/modes_j.jsonl
for f in gpurun_out/launch_dense_*.csv; do echo $f; python scripts/launch_summary.py $f; done
tail -n 5 gpurun_out/dense.err
