# final round-2 evidence: memcheck over the changed encode paths, GPU suite,
# smoke, bench lines, sweeps, ncu at bench size (TAG r02c), bench launch list
set -x
timeout 1800 compute-sanitizer --tool memcheck --print-limit 50 \
  python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_parity.py -q -x -k "dense or encode_decode or k3e or piece" > gpurun_out/memcheck_r02c.log 2>&1
tail -3 gpurun_out/memcheck_r02c.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload c4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python scripts/bench_modes.py > gpurun_out/modes.jsonl 2> gpurun_out/modes.err
timeout 900 python scripts/bench_dense.py > gpurun_out/dense.jsonl 2> gpurun_out/dense.err
timeout 600 python scripts/bench_paged.py > gpurun_out/paged.json 2> gpurun_out/paged.err
TAG=r02c bash scripts/gpu_prof_bench.sh > gpurun_out/prof_bench.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
for f in c2 c3 c4 ref; do tail -n 1 gpurun_out/bench_$f.json; done
