# round-end evidence: tests, smoke, bench lines (c2, c3, reference arm), launch
# list of the bench command and full ncu captures of the codec kernels
set -x
TAG=${TAG:-r01r}
bash scripts/gpu_round.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/launch_bench.log 2>&1
for f in bf16 e5m2; do
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'encode_tiles|decode_persistent' -s 2 -c 2 \
  -o gpurun_out/prof_${TAG}_$f python scripts/profile_kernels.py $f $((1<<28)) 2 > gpurun_out/prof_$f.log 2>&1
done
