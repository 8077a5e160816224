# dense stager walk (group merge, no K3e) vs K3e path
set -x
SZ_DEC_MARKED=2 timeout 900 python -m pytest tests/test_gpu_dense_escapes.py -x -q -k "stager" 2>&1 | tail -2 > gpurun_out/pytest_t.log
SZ_DENSE_PATHS=1,2 SZ_DENSE_RATES=0.03,0.0789 timeout 900 python scripts/bench_dense.py > gpurun_out/dense_t.jsonl 2> gpurun_out/dense.err
SZ_DEC_MARKED=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_walk_bf16.csv python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > /dev/null 2>&1
cat gpurun_out/pytest_t.log gpurun_out/dense_t.jsonl; python scripts/launch_summary.py gpurun_out/launch_walk_bf16.csv | grep decode
