# escape-dense decode profile (BF16 / E5M2 top-8 3-bit, 2^28): launch lists
# of both decoder paths and full captures of K4 + K3e on the K3e path
set -x
N=$((1<<28))
for path in 0 1; do
  SZ_DEC_MARKED=$path timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dense_p$path.csv python scripts/profile_kernels.py bf16 $N 2 3 > /dev/null 2>&1
  SZ_DEC_MARKED=$path timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launch_dense_e5_p$path.csv python scripts/profile_kernels.py e5m2 $N 2 3 > /dev/null 2>&1
done
SZ_DEC_MARKED=1 timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'decode_persistent|escape_marks' -s 2 -c 2 -o /tmp/dense_k3e python scripts/profile_kernels.py bf16 $N 2 3 > gpurun_out/prof_dense.log 2>&1
SZ_DEC_MARKED=1 timeout 900 ncu -f --set full --clock-control none --import-source on \
  -k regex:'decode_persistent' -s 1 -c 1 -o /tmp/dense_k3e_e5 python scripts/profile_kernels.py e5m2 $N 2 3 >> gpurun_out/prof_dense.log 2>&1
for r in dense_k3e dense_k3e_e5; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/raw_$r.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass -k regex:decode_persistent > gpurun_out/src_$r.csv 2>/dev/null
done
ncu -i /tmp/dense_k3e.ncu-rep --page source --csv --print-source sass -k regex:escape_marks > gpurun_out/src_marks.csv 2>/dev/null
cp /tmp/dense_k3e.ncu-rep gpurun_out/ 2>/dev/null
for f in gpurun_out/launch_dense_*.csv; do echo $f; python scripts/launch_summary.py $f; done
ls -la gpurun_out
