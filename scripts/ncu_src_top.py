"""Hottest SASS lines of an `ncu --page source --csv --print-source sass`
export (CPU): samples, top stall reasons, executed instructions.

usage: python scripts/ncu_src_top.py <source.csv> [top=30]
"""
import csv
import io
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lines = open(path).read().splitlines()
st = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[st:]))))
h = rows[0]
rows = [r for r in rows[1:] if r and r[0].startswith("0x")]
si, ni, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[si] or 0) for r in rows)
print(f"total samples {tot}, instructions {sum(int(r[ni] or 0) for r in rows)}")
order = sorted(range(len(rows)), key=lambda k: -int(rows[k][si] or 0))
for k in order[:top]:
    r = rows[k]
    st = sorted(((int(r[i] or 0), c[6:]) for i, c in cols), reverse=True)[:3]
    print(f"{k:5d} {int(r[si]):7d} {100 * int(r[si]) / tot:5.1f}%  ex={r[ni]:>9}  {r[src].strip()[:60]:60s} "
          + " ".join(f"{c}={v}" for v, c in st if v))
