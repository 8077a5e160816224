# ncu -f --set full of every codec kernel at the bench's own size (2^31 words,
# c2 BF16 and c3 E5M2), one launch each, so bench.py's roofline.traffic is a
# measurement of that launch, not a scaled smaller capture; plus the launch
# list of the bench command itself.  Reports are summarised on the box into
# gpurun_out/ (the .ncu-rep files stay in /tmp: too large to copy back).
set -x
TAG=${TAG:-r02a}
N=$((1<<31))
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/launch_bench.log 2>&1
for f in bf16 e5m2; do
  w=c2; [ $f = e5m2 ] && w=c3
  timeout 1200 ncu -f --set full --clock-control none --import-source on \
    -k regex:'encode_tiles|decode_persistent|escape_gather|escape_heavy|offsets_kernel|hist_kernel|pack_values' -c 14 \
    -o /tmp/prof_${TAG}_$f python scripts/profile_kernels.py $f $N 1 > gpurun_out/prof_$f.log 2>&1
  SZ_PROFILES_DIR=gpurun_out python scripts/ncu_summary.py /tmp/prof_${TAG}_$f.ncu-rep $N ${w}_$TAG $f \
    > /dev/null 2>> gpurun_out/prof_$f.log
  ncu -i /tmp/prof_${TAG}_$f.ncu-rep --page details --csv > gpurun_out/details_${TAG}_$f.csv 2>/dev/null
done
ls -la gpurun_out
