# Quick GPU validation of a kernel change: GPU parity suite, smoke, bench c2/c3.
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python scripts/profile_e2e.py > gpurun_out/e2e_phases.txt 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/e2e_phases.txt
python - <<'PY'
import json
for w in ("c2", "c3"):
    try:
        d = json.loads(open(f"gpurun_out/bench_{w}.json").read().strip().splitlines()[-1])
        print(w, "enc", d["encode_gbs"], "dec", d["decode_gbs"], "frac", d["roofline"]["encode_frac"], d["roofline"]["decode_frac"], "e2e", d["e2e"]["value"], d["clocks"])
    except Exception as e:
        print(w, "bench failed", e)
PY
