# fixed per-tile scratch (TILE/8 records) + values-only staging; K1 lane-column bins
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 900 python scripts/bench_modes.py "bf16 top16 explicit c1024" "bf16 top8 3-bit c1024" "e5m2 top16 explicit c1024" "e5m2 top8 3-bit c1024" "e4m3 top8 3-bit c1024" > gpurun_out/modes.jsonl 2> gpurun_out/modes.err
timeout 300 python bench.py --no-cpu-baseline --steps 10 --e2e-steps 1 > gpurun_out/f_c2.json 2>/dev/null
timeout 300 python bench.py --workload c3 --no-cpu-baseline --steps 10 --e2e-steps 1 > gpurun_out/f_c3.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_3bit.csv python scripts/profile_kernels.py bf16 268435456 2 3 > /dev/null 2>&1
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:encode_tiles -s 1 -c 1 -o /tmp/enc3 python scripts/profile_kernels.py bf16 268435456 1 3 > /dev/null 2>&1
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:encode_tiles -s 1 -c 1 -o /tmp/enc4 python scripts/profile_kernels.py bf16 268435456 1 4 > /dev/null 2>&1
for r in enc3 enc4; do ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/raw_$r.csv 2>/dev/null; ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$r.csv 2>/dev/null; done
cat gpurun_out/pytest_gpu.log gpurun_out/modes.jsonl
python - <<'P'
import json
for f in ['f_c2','f_c3']:
    d=json.loads(open('gpurun_out/'+f+'.json').read().strip().splitlines()[-1]); print(f, d['encode_gbs'], d['decode_gbs'], d['calibration_histogram_gbs'])
P
python scripts/launch_summary.py gpurun_out/launches_3bit.csv
ls -la gpurun_out
