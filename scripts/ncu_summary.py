"""Summarise ncu reports into profiles/ (markdown table + per-element traffic JSON).

usage: python scripts/ncu_summary.py <report.ncu-rep> <n_elements> <tag> [fmt]
Writes profiles/ncu_<tag>.md and profiles/ncu_traffic_<tag>.json.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_inst"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}


def main():
    rep, n, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    word_bytes = 2 if (len(sys.argv) < 5 or sys.argv[4] == "bf16") else 1
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kernels = []
    for d in data:
        k = {"kernel": d[hdr.index("Kernel Name")].split("(")[0]}
        for m, key in METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = float(d[i].replace(",", "")) if d[i] not in ("", "n/a") else None
            if v is not None and units[i] in SCALE:
                v *= SCALE[units[i]]
            k[key] = v
        kernels.append(k)
    lines = [f"# ncu --set full summary: {Path(rep).name}",
             "",
             f"Workload: {n} elements ({n * word_bytes / 2**20:.0f} MiB of words), "
             "scripts/profile_kernels.py, one launch per kernel after warm-up, "
             "`--clock-control none` (cold-cache replays: compare shares, not absolutes).",
             "",
             "| kernel | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM B/elem | DRAM % peak | "
             "issue % | ALU % | regs | grid x block |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic, absolute = {}, {}
    for k in kernels:
        tot = (k.get("dram_read") or 0) + (k.get("dram_write") or 0)
        lines.append(
            f"| {k['kernel']} | {k['time'] * 1e6:.1f} | {k['dram_read'] / 1e6:.1f} | "
            f"{k['dram_write'] / 1e6:.1f} | {tot / n:.4f} | {k.get('dram_pct', 0):.1f} | "
            f"{k.get('issue_pct', 0):.1f} | {k.get('alu_pct', 0):.1f} | {k.get('regs', 0):.0f} | "
            f"{k.get('grid', 0):.0f} x {k.get('block', 0):.0f} |")
        name = re.sub(r"^void ", "", k["kernel"]).split("<")[0].split("::")[-1]
        traffic.setdefault(name, tot / n)
        absolute.setdefault(name, int(tot))
    # SZ_PROFILES_DIR: write elsewhere (on the GPU box: gpurun_out/, which
    # comes back; the .ncu-rep files themselves may be too large to)
    out_dir = Path(os.environ.get("SZ_PROFILES_DIR", ROOT / "profiles"))
    out_dir.mkdir(exist_ok=True)
    (out_dir / f"ncu_{tag}.md").write_text("\n".join(lines) + "\n")
    (out_dir / f"ncu_traffic_{tag}.json").write_text(json.dumps(
        {"source": Path(rep).name, "n_elements_profiled": n,
         "dram_bytes_per_element": traffic, "dram_bytes_per_launch": absolute},
        indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
