# round-2 evidence after the K3e/K4-stager changes (TAG r02e): memcheck and
# racecheck over the escape-dense paths, GPU suite, smoke, bench lines,
# sweeps, launch lists of the K3e path
set -x
timeout 1800 compute-sanitizer --tool memcheck --print-limit 50 \
  python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_robustness.py -q -x > gpurun_out/memcheck_r02e.log 2>&1
tail -3 gpurun_out/memcheck_r02e.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 \
  python -m pytest tests/test_gpu_dense_escapes.py -q -x -k "roundtrip" > gpurun_out/racecheck_r02e.log 2>&1
tail -3 gpurun_out/racecheck_r02e.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload c4 --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python scripts/bench_modes.py > gpurun_out/modes.jsonl 2> gpurun_out/modes.err
timeout 900 python scripts/bench_dense.py > gpurun_out/dense.jsonl 2> gpurun_out/dense.err
for f in bf16 e5m2; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/dense_k3e_${f}_r02e.csv python scripts/profile_kernels.py $f $((1<<28)) 2 3 > /dev/null 2>&1
done
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
for f in c2 c3 c4 ref; do tail -n 1 gpurun_out/bench_$f.json | cut -c1-400; done
