# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_small.py
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize_small.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize ok' gpurun_out/sanitize_$t.log | tr '\n' ' ')"
done
