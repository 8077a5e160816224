# E5M2 3-bit K2a with 7 writers: GPU suite + mode sweep
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 900 python scripts/bench_modes.py > gpurun_out/modes.jsonl 2> gpurun_out/modes.err
cat gpurun_out/pytest_gpu.log gpurun_out/modes.jsonl
