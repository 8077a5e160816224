# ncu evidence for the current kernels: launch list of a short bench run,
# full captures of the codec kernels (BF16 and E5M2, 2^28 words), PCIe probe.
set -x
TAG=${TAG:-r01e}
python scripts/pcie_probe.py > gpurun_out/pcie.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
  > gpurun_out/launch_bench.log 2>&1
for f in bf16 e5m2; do
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'encode_tiles|decode_persistent|escape_gather|offsets_kernel|hist_kernel' -s 5 -c 6 \
  -o gpurun_out/prof_${TAG}_$f python scripts/profile_kernels.py $f $((1<<28)) 3 > gpurun_out/prof_$f.log 2>&1
done
ls -la gpurun_out; cat gpurun_out/pcie.txt
