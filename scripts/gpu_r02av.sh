# K3e: failed checks accumulate per lane and send the window through the
# exact walk (base) vs a branch per round (k3ebranch); parity first
set -x
rm -f gpurun_out/ab.txt
timeout 900 python -m pytest tests/test_gpu_dense_escapes.py tests/test_gpu_robustness.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
VARIANTS="base k3ebranch" CONFIGS='"bf16 top8 3-bit c1024" "e5m2 top8 3-bit c1024"' bash scripts/ab_variants.sh
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv -k regex:escape_marks \
    --log-file gpurun_out/k3e_av.csv python scripts/profile_kernels.py e5m2 $((1<<28)) 2 3 > /dev/null 2>&1
grep escape_marks gpurun_out/k3e_av.csv | tail -4 | cut -d, -f5,13-
