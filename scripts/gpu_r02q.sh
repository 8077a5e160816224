# E5M2 decode addressing (PRMT + IMAD) A/B against the numbers of r02o; handoff piece-size sweep
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense_escapes.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_q.log
timeout 600 python scripts/bench_modes.py "e5m2 top16 explicit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c1024" > gpurun_out/modes_q.jsonl 2>/dev/null
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null
for pc in 26 27; do
  timeout 600 python scripts/bench_handoff.py --loopback --reps 3 --piece $((1<<pc)) > gpurun_out/handoff_p$pc.json 2>/dev/null
done
cat gpurun_out/pytest_q.log gpurun_out/modes_q.jsonl gpurun_out/bench_c3.json gpurun_out/handoff_p*.json
