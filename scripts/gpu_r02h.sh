# K3e escape-dense decode: GPU tests of the dense / parity / robustness suites, rate sweep, modes
set -x
timeout 1500 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_parity.py tests/test_gpu_robustness.py -x -q 2>&1 | tail -15 > gpurun_out/pytest_k3e.log
timeout 900 python scripts/bench_dense.py > gpurun_out/dense.jsonl 2> gpurun_out/dense.err
timeout 600 python scripts/bench_modes.py "bf16 top16 explicit c1024" "bf16 top8 3-bit c1024" "e5m2 top16 explicit c1024" "e5m2 top8 3-bit c1024" "e4m3 top8 3-bit c1024" > gpurun_out/modes_h.jsonl 2> gpurun_out/modes_h.err
cat gpurun_out/pytest_k3e.log gpurun_out/dense.jsonl gpurun_out/modes_h.jsonl; tail -5 gpurun_out/dense.err gpurun_out/modes_h.err
