# per-role K2a cycle counters after the 7-writer change (E5M2 / BF16, 3-bit)
set -x
rm -f gpurun_out/timers.txt
for cfg in "e5m2 268435456 1 3" "bf16 268435456 1 3" "e5m2 268435456 1 4"; do
  echo "== $cfg" >> gpurun_out/timers.txt
  SZ_LIB_VARIANT=timers SZ_DEBUG_TIMERS=1 timeout 300 python scripts/profile_kernels.py $cfg 2>&1 | grep timers | tail -1 >> gpurun_out/timers.txt
done
cat gpurun_out/timers.txt
