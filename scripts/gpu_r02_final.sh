# round-2 evidence: GPU suite, smoke, bench lines c2 / c3 / c4 / reference arm,
# mode sweep, escape-rate sweep, launch list of the bench command
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload c4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python scripts/bench_modes.py > gpurun_out/modes.jsonl 2> gpurun_out/modes.err
timeout 900 python scripts/bench_dense.py > gpurun_out/dense.jsonl 2> gpurun_out/dense.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r02b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench_c2.json gpurun_out/bench_c3.json gpurun_out/bench_c4.json gpurun_out/bench_ref.json
python scripts/launch_summary.py gpurun_out/launches_r02b.csv | head -12
for f in gpurun_out/*.err; do echo $f; tail -n 3 $f; done
