"""Summarise an ncu report: headline metrics and the hottest SASS lines with
their CUDA source line (reads `ncu -i REP --page source --print-source=cuda,sass`)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy",
        "Registers Per Thread", "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction", "Issue Slots Busy",
        "Dynamic Shared Memory Per Block")
want += ("Executed Ipc Active", "No Eligible", "Eligible Warps Per Scheduler", "Shared Memory Configuration Size",
         "Theoretical Occupancy", "Block Limit Shared Mem", "Block Limit Registers")
cols = None
for row in csv.reader(det.splitlines()):
    if "Metric Name" in row:
        cols = (row.index("Metric Name"), row.index("Metric Unit"), row.index("Metric Value"))
        continue
    if cols and len(row) > cols[2] and row[cols[0]] in want:
        print(f"{row[cols[0]]:40s} {row[cols[2]]:>12s} {row[cols[1]]}")
mix = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(mix.splitlines()))
hdr = None
cur_line = ""
samples = []
for r in rows:
    if len(r) >= 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:
        cur_line = f"{r[0]}: {r[1].strip()[:70]}"
        continue
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    samples.append((s, cur_line, r[3].strip()[:50]))
tot = sum(s for s, _, _ in samples) or 1
by_line = {}
for s, ln, _ in samples:
    by_line[ln] = by_line.get(ln, 0) + s
print(f"\n== top source lines by warp-stall samples (total {tot:.0f})")
for ln, s in sorted(by_line.items(), key=lambda x: -x[1])[:top]:
    print(f"{100 * s / tot:5.1f}%  {ln}")
