"""Summarise an ncu report: headline metrics, stall reasons and opcode mix (reads the .ncu-rep here)."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy",
        "Executed Ipc Active", "Warp Cycles Per Issued Instruction", "No Eligible", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "DRAM Throughput", "Dynamic Shared Memory Per Block", "L1/TEX Hit Rate"]
rows_d = list(csv.reader(io.StringIO(det)))
hd = {h: i for i, h in enumerate(rows_d[0])}
for r in rows_d[1:]:
    if len(r) > hd["Metric Value"] and r[hd["Metric Name"]] in keys:
        print(f"{r[hd['Metric Name']]:40s} {r[hd['Metric Value']]} {r[hd['Metric Unit']]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stall = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
ops = Counter()
inst = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    for h in stall:
        try:
            tot[h] += int(r[idx[h]])
        except ValueError:
            pass
    try:
        n = int(r[idx["Instructions Executed"]])
    except ValueError:
        continue
    inst += n
    t = r[idx["Source"]].split()
    if t:
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += n
s = sum(tot.values())
print("stalls:", ", ".join(f"{h[6:]} {v / s * 100:.1f}%" for h, v in tot.most_common(8)))
print("SASS lines", len(rows) - 2, " warp instructions", inst)
print("opcodes:", ", ".join(f"{o} {v / inst * 100:.1f}%" for o, v in ops.most_common(14)))
