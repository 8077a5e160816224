# full GPU suite + mode sweep + escape-heavy + launch list of the 3-bit heavy config
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; tail -3 gpurun_out/pt_all.log
timeout 900 python scripts/bench_modes.py > gpurun_out/modes_all.jsonl 2>&1; cat gpurun_out/modes_all.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/modes_o.csv python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > /dev/null 2>&1
bash scripts/gpu_heavy.sh
