"""Aggregate ncu per-instruction stall samples by CUDA source line.

usage: python tools/sass_lines.py <report.ncu-rep> <kernel-substring> <lib.so> [topN]
Maps SASS offsets of the ncu source page to source lines via nvdisasm -g.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, kname, so = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    fname = sys.argv[5] if len(sys.argv) > 5 else kname  # function-name pattern in the disassembly
    # optional: attribute each instruction to the innermost frame inside this source file
    # (e.g. dt_kernel.cuh, so arithmetic helpers count at their call sites)
    focus = sys.argv[6] if len(sys.argv) > 6 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", f"regex:{kname}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0][0], 16)
    samples = {int(r[0], 16) - base: (float(r[ix["Warp Stall Sampling (All Samples)"]] or 0),
                                     float(r[ix["Instructions Executed"]] or 0), r[1].strip(),
                                     {k: float(r[ix[k]] or 0) for k in hdr if k.startswith("stall_") and "Not Issued" not in k})
               for r in data}
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
    dis = ""
    for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
        d = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
        if re.search(r"\.text\.\S*" + re.escape(fname.split("|")[0]), d):
            dis = d
            break
    # find function section by mangled-name match
    lines = dis.splitlines()
    cur_fn, cur_line, in_fn, prev_marker, focus_hit = None, None, False, False, False
    addr_line = {}
    for ln in lines:
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            in_fn = fname.replace("<", "").split("(")[0] in m.group(1) or all(p in m.group(1) for p in fname.split("|"))
            continue
        if not in_fn:
            continue
        # an inline chain is a run of markers, innermost first: keep the first of each run
        m = re.search(r"//## File \"(.*?)\", line (\d+)", ln)
        if m:
            loc = (os.path.basename(m.group(1)), int(m.group(2)))
            if not prev_marker:
                cur_line = loc
                focus_hit = focus is not None and loc[0] == focus
            elif focus is not None and not focus_hit and loc[0] == focus:
                cur_line = loc
                focus_hit = True
            prev_marker = True
            continue
        prev_marker = False
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_line:
            addr_line[int(m.group(1), 16)] = cur_line
    agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
    tot = 0.0
    for off, (s, ex, src, st) in samples.items():
        key = addr_line.get(off, ("?", 0))
        agg[key][0] += s
        agg[key][1] += ex
        agg[key][2].update(st)
        tot += s
    print(f"total samples {tot:.0f}, mapped offsets {sum(1 for o in samples if o in addr_line)}/{len(samples)}")
    for key, (s, ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        tops = ", ".join(f"{k[6:]}={v/s*100:.0f}%" for k, v in st.most_common(3) if s)
        print(f"{key[0]}:{key[1]:5d}  {100*s/tot:5.1f}%  inst={ex:.3g}  [{tops}]")


if __name__ == "__main__":
    main()
