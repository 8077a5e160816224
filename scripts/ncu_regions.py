"""Stall-reason breakdown of one kernel's SASS, split into address ranges.

usage: python scripts/ncu_regions.py <report> <kernel regex> [block=80] [min_samples=300]
Prints per block of SASS instructions: executed instructions, samples and
the top stall reasons, so warp roles (producer / stagers / workers) can be
told apart by their code ranges.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 80
mins = int(sys.argv[4]) if len(sys.argv) > 4 else 300
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
lines = out.splitlines()
st = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[st:]))))
h = rows[0]
end = next((i for i, r in enumerate(rows[1:], 1) if r and r[0] in ("Address", "Kernel Name")), len(rows))
rows = rows[1:end]
ni, si, src = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = [h.index(c) for c in cols]
tot = sum(int(r[si] or 0) for r in rows)
print(f"total samples {tot}")
for b in range(0, len(rows), blk):
    part = rows[b:b + blk]
    s = sum(int(r[si] or 0) for r in part)
    if s < mins:
        continue
    n = sum(int(r[ni] or 0) for r in part)
    st_ = {c[6:]: sum(int(r[i] or 0) for r in part) for c, i in zip(cols, idx)}
    topr = " ".join(f"{k}={v}" for k, v in sorted(st_.items(), key=lambda x: -x[1])[:4])
    print(f"[{b:5d}-{b + blk - 1:5d}] inst {n:11d} samp {s:6d} ({100 * s / tot:4.1f}%) {topr} | {part[0][src][:40]}")
