# full GPU suite + mode sweep + launch list of the 3-bit heavy config
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; tail -3 gpurun_out/pt_all.log
timeout 900 python scripts/bench_modes.py > gpurun_out/modes_all.jsonl 2>&1; cat gpurun_out/modes_all.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/modes_n.csv python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'escape_heavy|encode_tiles' -s 2 -c 2 -o gpurun_out/prof_r01n_heavy python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > gpurun_out/prof_heavy.log 2>&1
