"""Per-kernel device time from an ncu launch list (gpu__time_duration.sum CSV).

usage: python scripts/launch_summary.py <launches.csv> [skip_regex]
"""
import csv
import re
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
skip = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows:
    name = r[4].split("(")[0].replace("void ", "")
    if skip and skip.search(name):
        continue
    val = float(r[14].replace(",", ""))
    us = {"nsecond": val / 1000.0, "usecond": val, "msecond": val * 1000.0}.get(r[13], val / 1000.0)
    tot[name] += us
    cnt[name] += 1
all_us = sum(tot.values())
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"{tot[k] / cnt[k]:10.1f} us x{cnt[k]:3d}  {100 * tot[k] / all_us:5.1f}%  {k}")
