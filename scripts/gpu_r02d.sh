set -x
timeout 600 python -m pytest tests/test_gpu_realkv.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_realkv.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err
TAG=r02a bash scripts/gpu_prof_bench.sh
cat gpurun_out/pytest_realkv.log gpurun_out/bench_c2.json gpurun_out/bench_ref.json
