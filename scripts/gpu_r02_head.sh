# re-entry check of HEAD on a fresh box: GPU suite, smoke, default bench line, c3 line
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/pytest_gpu_head.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_head.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_head_c2.json 2> gpurun_out/bench_head_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_head_c3.json 2> gpurun_out/bench_head_c3.err
cat gpurun_out/pytest_gpu_head.log gpurun_out/smoke_head.log
tail -n 1 gpurun_out/bench_head_c2.json | cut -c1-400
tail -n 1 gpurun_out/bench_head_c3.json | cut -c1-400
