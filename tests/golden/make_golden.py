"""Regenerates tests/golden/affine_decay.json from the reference's own golden
files (run in the build container, where /root/reference exists):

  /root/reference/proj/data/affine_decay_net.json   the 2-D affine net
  /root/reference/proj/data/affine_decay_golden.csv `reach-dt --x0-center 0.5,0.5
                                                    --eps 0.125 --steps 8` output
                                                    (test_cli.cpp:43-49)

The fixture re-encodes them (net params, X0, and the expected boxes as exact
hex floats) so the tests need nothing from /root/reference at run time.
"""
import csv
import json
import os
import sys

REF = "/root/reference/proj/data"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "affine_decay.json")


def main():
    net = json.load(open(os.path.join(REF, "affine_decay_net.json")))
    layers = []
    for L in net["layers"]:
        layers.append({"act": L["act"], "w": L["w"], "b": L["b"]})
    rows = list(csv.DictReader(open(os.path.join(REF, "affine_decay_golden.csv"))))
    steps = 1 + max(int(r["step"]) for r in rows)
    n = 1 + max(int(r["dim"]) for r in rows)
    lo = [[None] * n for _ in range(steps)]
    hi = [[None] * n for _ in range(steps)]
    text = {}
    for r in rows:
        k, d = int(r["step"]), int(r["dim"])
        lo[k][d] = float(r["lo"]).hex()
        hi[k][d] = float(r["hi"]).hex()
        text[f"{k},{d}"] = [r["lo"], r["hi"]]
    fx = {
        "source": "reference proj/data/affine_decay_{net.json,golden.csv}; reach-dt --x0-center 0.5,0.5 --eps 0.125 --steps 8",
        "layers": layers,
        "x0_center": [0.5, 0.5],
        "eps": 0.125,
        "horizon": steps - 1,
        "n": n,
        "m": 0,
        "expected_lo_hex": lo,
        "expected_hi_hex": hi,
        "expected_csv_text": text,
    }
    json.dump(fx, open(OUT, "w"), indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    sys.exit(main())
