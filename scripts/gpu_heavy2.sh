# parity + escape-heavy profile (decode) + mode sweep of the heavy / c256 modes
set -x
TAG=${TAG:-r01k}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paged.py tests/test_gpu_container.py -x -q > gpurun_out/pt_heavy.log 2>&1; tail -3 gpurun_out/pt_heavy.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/modes_k.csv python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'decode_persistent|escape_heavy' -s 2 -c 2 -o gpurun_out/prof_${TAG}_heavy python scripts/profile_kernels.py bf16 $((1<<28)) 2 3 > gpurun_out/prof_heavy.log 2>&1
timeout 900 python scripts/bench_modes.py "bf16 top16 explicit c1024" "bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024" "bf16 top16 explicit c256" "e4m3 top8 3-bit c1024" "e5m2 top16 explicit c1024"
