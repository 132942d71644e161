"""Summarise an ncu report: duration, stall reasons, top SASS lines by stall samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
for row in csv.reader(io.StringIO(det)):
    if len(row) > 12 and row[12] in ("Duration", "Registers Per Thread", "Grid Size", "Block Size",
                                      "DRAM Throughput", "Warp Cycles Per Issued Instruction", "Issued Ipc Active",
                                      "L2 Hit Rate", "Achieved Occupancy"):
        print(f"{row[12]:40s} {row[14]} {row[13]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {r: h.index(r) for r in reasons}
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = {r: sum(float(x[idx[r]] or 0) for x in data) for r in reasons}
T = sum(tot.values()) or 1
print("stalls:", ", ".join(f"{r[6:]} {100 * v / T:.1f}%" for r, v in sorted(tot.items(), key=lambda x: -x[1]) if v / T > 0.01))
TT = sum(float(x[iall] or 0) for x in data) or 1
for r in sorted(data, key=lambda x: -float(x[iall] or 0))[:top]:
    why = max(reasons, key=lambda k: float(r[idx[k]] or 0))
    print(f"{100 * float(r[iall]) / TT:5.1f}% {r[ia][-5:]} {why[6:]:16s} {r[isrc][:80]}")
