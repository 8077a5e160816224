# racecheck + synccheck over the final decoder (T12, 3 CTAs/SM) and encoder (K2b word copies, K6)
set -x
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 \
  python -m pytest tests/test_gpu_dense_escapes.py -q -x -k "roundtrip" > gpurun_out/racecheck_r02d.log 2>&1
tail -3 gpurun_out/racecheck_r02d.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 \
  python -m pytest tests/test_gpu_dense_escapes.py -q -x -k "roundtrip" > gpurun_out/synccheck_r02d.log 2>&1
tail -3 gpurun_out/synccheck_r02d.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 \
  python scripts/sanitize_small.py > gpurun_out/racecheck_small_r02d.log 2>&1
tail -3 gpurun_out/racecheck_small_r02d.log
