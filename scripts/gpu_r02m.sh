# per-role K2a cycle counters (SZ_TIMERS variant) for escape-dense and realistic books
set -x
for cfg in "e5m2 268435456 1 3" "bf16 268435456 1 3" "e5m2 268435456 1 4" "bf16 268435456 1 4"; do
  echo "== $cfg" >> gpurun_out/timers.txt
  SZ_LIB_VARIANT=timers SZ_DEBUG_TIMERS=1 timeout 300 python scripts/profile_kernels.py $cfg 2>&1 | grep timers | tail -2 >> gpurun_out/timers.txt
done
cat gpurun_out/timers.txt
