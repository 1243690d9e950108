"""Turn a gpurun_out/<tag>/ capture into committed evidence under profiles/:
the ncu launch list, per-capture key metrics (details page) and raw metric
CSVs, plus a markdown summary."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

run = sys.argv[1]
tag = sys.argv[2]
out = os.path.join("profiles", tag)
os.makedirs(out, exist_ok=True)
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Elapsed Cycles", "SM Active Cycles",
        "Issue Slots Busy", "Registers Per Thread", "Grid Size", "Achieved Occupancy", "L2 Hit Rate",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
md = [f"# ncu evidence {tag}", "", f"Source run: `{run}` (B200, `--clock-control none`).", ""]
for f in sorted(os.listdir(run)):
    p = os.path.join(run, f)
    if f.endswith(".ncu-rep"):
        name = f[:-8]
        det = subprocess.run(["ncu", "-i", p, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        raw = subprocess.run(["ncu", "-i", p, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        with open(os.path.join(out, name + "_raw.csv"), "w") as fh:
            fh.write(raw)
        rows = list(csv.reader(io.StringIO(det)))
        kname = rows[1][4] if len(rows) > 1 and len(rows[1]) > 4 else name
        md.append(f"## {name}")
        md.append(f"Kernel: `{kname[:160]}`")
        md.append("")
        md.append("| metric | value |")
        md.append("|---|---|")
        seen = set()
        for r in rows[1:]:
            if len(r) >= 4 and r[-3] in KEYS and r[-3] not in seen:
                seen.add(r[-3])
                md.append(f"| {r[-3]} ({r[-2]}) | {r[-1]} |")
        rr = list(csv.reader(io.StringIO(raw)))
        if len(rr) >= 3:
            h, units, v = rr[0], rr[1], rr[-1]
            for k in RAW:
                if k in h:
                    i = h.index(k)
                    md.append(f"| {k} ({units[i]}) | {v[i]} |")
        md.append("")
    elif f.endswith(".csv") and "launch" in f:
        shutil.copy(p, os.path.join(out, f))
        s = subprocess.run([sys.executable, "scripts/launch_stats.py", p], capture_output=True, text=True).stdout
        md += ["## launch list (TWO solves -- scripts/one_solve.py runs one warm-up and one timed solve -- plus setup; cold-cache, serialised: divide the counts by 2 per solve)", "", "```", s.strip(), "```", ""]
    elif f.endswith(".json") or f.endswith(".txt"):
        shutil.copy(p, os.path.join(out, f))
with open(os.path.join(out, "SUMMARY.md"), "w") as fh:
    fh.write("\n".join(md) + "\n")
print("wrote", out)
