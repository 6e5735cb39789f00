"""Per-kernel share of device time from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg, cnt = defaultdict(float), defaultdict(int)
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
for r in rows:
    if "Kernel Name" in r:
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and len(r) == len(hdr) and r[hdr["Metric Name"]] == "gpu__time_duration.sum":
        k = r[hdr["Kernel Name"]].split("(")[0]
        agg[k] += float(r[hdr["Metric Value"]].replace(",", "")) * scale.get(r[hdr["Metric Unit"]], 1.0)
        cnt[k] += 1
tot = sum(agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"| {k} | {cnt[k]} | {v:.2f} ms | {v / tot * 100:.1f}% |")
