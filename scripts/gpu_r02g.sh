# round-2 re-entry: GPU tests, smoke, bench lines (c2 / c3 / reference), mode sweep
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err
timeout 900 python scripts/bench_modes.py > gpurun_out/modes.jsonl 2> gpurun_out/modes.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cat gpurun_out/bench_c2.json gpurun_out/bench_c3.json gpurun_out/bench_ref.json gpurun_out/modes.jsonl; for f in gpurun_out/*.err; do tail -n 5 "$f"; done
