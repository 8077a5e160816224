# round-2 closing evidence (TAG r02f, after K2b's two-records-per-lane path):
# GPU suite, smoke, bench lines c2 / c3 / c4 / reference arm, mode sweep,
# then ncu at the bench's size + the bench launch list (gpu_prof_bench.sh)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu_r02f.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_r02f_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_r02f_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload c4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_r02f_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r02f_reference.json 2> gpurun_out/bench_ref.err
timeout 900 python scripts/bench_modes.py > gpurun_out/bench_modes_r02i.jsonl 2> gpurun_out/modes.err
TAG=r02f bash scripts/gpu_prof_bench.sh > gpurun_out/prof_bench.log 2>&1
cat gpurun_out/pytest_gpu_r02f.log gpurun_out/smoke.log
for f in c2 c3 c4 reference; do tail -n 1 gpurun_out/bench_r02f_$f.json | cut -c1-300; done
