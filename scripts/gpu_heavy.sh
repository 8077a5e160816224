timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paged.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --escape-rate 0.0789 --steps 5 --warmup 3 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 eps7.89 enc', d['encode_gbs'], 'dec', d['decode_gbs'], 'ratio', d['compression_ratio'])"
timeout 300 python bench.py --workload c3 --no-cpu-baseline --escape-rate 0.0789 --steps 5 --warmup 3 --e2e-steps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 eps7.89 enc', d['encode_gbs'], 'dec', d['decode_gbs'], 'ratio', d['compression_ratio'])"
timeout 300 python scripts/bench_handoff.py --loopback 2>&1 | tail -1
