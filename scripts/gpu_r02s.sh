# crossover sweep after the branch-free merge
set -x
SZ_DENSE_RATES=0.008,0.012,0.016,0.02,0.024,0.03 timeout 900 python scripts/bench_dense.py > gpurun_out/dense_s.jsonl 2> gpurun_out/dense.err
cat gpurun_out/dense_s.jsonl
