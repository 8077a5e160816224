"""Top stalled SASS instructions of one kernel in an ncu report (source page).

usage: python scripts/ncu_hot.py <report> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
# keep the first kernel instance only (later ones repeat the header)
end = next((i for i, r in enumerate(rows[1:], 1) if r and r[0] in ("Address", "Kernel Name")),
           len(rows))
rows = rows[:end]
si, ni, src = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
data = [(int(r[si] or 0), int(r[ni] or 0), r[src].strip(), i) for i, r in enumerate(rows[1:]) if len(r) > max(si, ni, src)]
tot = sum(d[0] for d in data)
print(f"total samples {tot}")
for s, n, t, i in sorted(data, reverse=True)[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}% {n:10d}  [{i:5d}] {t}")
