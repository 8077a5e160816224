timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/handoff_launches.csv python scripts/bench_handoff.py --loopback --elems $((1<<27)) --reps 1 > /dev/null 2>&1
python - <<'PY'
import csv
lines=open('gpurun_out/handoff_launches.csv').read().splitlines()
i=[j for j,l in enumerate(lines) if l.startswith('"ID"')][0]
rows=list(csv.reader(lines[i:]))
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value")
from collections import defaultdict
d=defaultdict(list)
for r in rows[1:]:
    d[r[ki].split('(')[0][:50]].append(float(r[vi].replace(',',''))/1e3)
for k,v in sorted(d.items(), key=lambda kv:-sum(kv[1])): print(f"{k:50s} n={len(v):4d} total={sum(v):9.1f}us mean={sum(v)/len(v):8.1f} max={max(v):8.1f}")
PY
