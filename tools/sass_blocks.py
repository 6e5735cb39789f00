"""Per-basic-block view of an ncu SASS source page: executed instructions,
stall samples (top reasons) and an opcode signature per block, hottest first.

usage: python tools/sass_blocks.py <report.ncu-rep> [kernel-regex] [topN]
"""
import collections
import csv
import subprocess
import sys


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else "dt_horizon"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", f"regex:{kre}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0][0], 16)
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    blocks = []
    cur = None
    for r in data:
        off = int(r[0], 16) - base
        src = r[1].strip()
        ex = float(r[ix["Instructions Executed"]] or 0)
        smp = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        if cur is None or (cur["ex"] and abs(ex - cur["ex_first"]) > 0.02 * max(ex, cur["ex_first"])):
            cur = {"start": off, "n": 0, "ex": 0.0, "ex_first": ex, "smp": 0.0, "ops": collections.Counter(),
                   "st": collections.Counter()}
            blocks.append(cur)
        cur["n"] += 1
        cur["ex"] += ex
        cur["smp"] += smp
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        cur["ops"][op.split(".")[0]] += 1
        for h in stall_cols:
            cur["st"][h[6:]] += float(r[ix[h]] or 0)
        cur["end"] = off
    tot_s = sum(b["smp"] for b in blocks)
    tot_e = sum(b["ex"] for b in blocks)
    print(f"total samples {tot_s:.0f}  executed {tot_e:.3g}")
    for b in sorted(blocks, key=lambda b: -b["smp"])[:top]:
        ops = " ".join(f"{k}{v}" for k, v in b["ops"].most_common(7))
        st = ", ".join(f"{k}={100*v/max(b['smp'],1):.0f}%" for k, v in b["st"].most_common(4))
        print(f"[{b['start']:#07x}-{b['end']:#07x}] n={b['n']:4d} smp={100*b['smp']/tot_s:5.1f}% "
              f"ex={100*b['ex']/tot_e:5.1f}% x{b['ex_first']:.3g}  {ops}\n      {st}")


if __name__ == "__main__":
    main()
