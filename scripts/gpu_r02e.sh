# escape-pool K2a: full GPU suite, escape-dense sweep, bench-size ncu
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 900 python scripts/bench_modes.py "bf16 top16 explicit c1024" "bf16 top8 3-bit c1024" "e5m2 top16 explicit c1024" "e5m2 top8 3-bit c1024" "e4m3 top8 3-bit c1024" > gpurun_out/modes.jsonl 2> gpurun_out/modes.err
timeout 300 python bench.py --no-cpu-baseline --escape-rate 0.0789 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/heavy_c2.json 2>/dev/null
timeout 300 python bench.py --workload c3 --no-cpu-baseline --escape-rate 0.0789 --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/heavy_c3.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_3bit.csv python scripts/profile_kernels.py bf16 268435456 2 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_3bit_e5.csv python scripts/profile_kernels.py e5m2 268435456 2 3 > /dev/null 2>&1
TAG=r02b bash scripts/gpu_prof_bench.sh
cat gpurun_out/pytest_gpu.log gpurun_out/modes.jsonl; tail -3 gpurun_out/modes.err
python scripts/launch_summary.py gpurun_out/launches_3bit.csv; python scripts/launch_summary.py gpurun_out/launches_3bit_e5.csv
