# memcheck over the K3e path (robustness harness forced through K3e + dense
# suites) and the loopback handoff launch list
set -x
timeout 1800 compute-sanitizer --tool memcheck --print-limit 50 \
  python -m pytest tests/test_gpu_robustness.py tests/test_gpu_dense_escapes.py -q -x -k "k3e" > gpurun_out/memcheck_k3e.log 2>&1
tail -4 gpurun_out/memcheck_k3e.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 \
  python -m pytest tests/test_gpu_dense_escapes.py -q -x -k "k3e and roundtrip" > gpurun_out/racecheck_k3e.log 2>&1
tail -4 gpurun_out/racecheck_k3e.log
bash scripts/gpu_handoff_prof.sh > gpurun_out/handoff_launch_summary.txt 2>&1
cat gpurun_out/handoff_launch_summary.txt
