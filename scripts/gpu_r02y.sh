# ncu source capture of the K3e K4 (E5M2 and BF16 top-8 3-bit)
set -x
for f in e5m2 bf16; do
SZ_DEC_MARKED=1 timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'decode_persistent' -s 1 -c 1 -o gpurun_out/k4k3e_$f python scripts/profile_kernels.py $f $((1<<28)) 2 3 > /dev/null 2>&1
done
ls -la gpurun_out
