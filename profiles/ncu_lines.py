"""Aggregate an ncu `--page source --csv --print-source=cuda,sass` export by CUDA source line:
warp-stall samples (total and top reasons) and executed instructions per line.
  ncu -i rep.ncu-rep --page source --csv --print-source=cuda,sass > x.csv; python ncu_lines.py x.csv"""
import csv
import sys
from collections import defaultdict


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r[:2] == ["Line No", "Source"])
    hdr = rows[hdr_i]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_ie = hdr.index("Instructions Executed")
    stall_cols = [(k, c) for k, c in enumerate(hdr) if c.startswith("stall_") and "Not Issued" not in c]
    src = {}
    agg = defaultdict(lambda: defaultdict(float))
    line = None
    fname = ""
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) < len(hdr) or r[0] == "Line No":
            continue
        if r[0].strip():
            line = (fname, int(r[0]))
            src[line] = r[1]
        if line is None:
            continue
        def f(x):
            try:
                return float(x)
            except ValueError:
                return 0.0
        agg[line]["samples"] += f(r[i_s])
        agg[line]["inst"] += f(r[i_ie])
        for k, c in stall_cols:
            agg[line][c] += f(r[k])
    tot = sum(a["samples"] for a in agg.values()) or 1.0
    print(f"total stall samples {tot:.0f}")
    for ln, a in sorted(agg.items(), key=lambda x: -x[1]["samples"])[:top]:
        reasons = sorted(((c[6:], v) for c, v in a.items() if c.startswith("stall_")), key=lambda x: -x[1])[:3]
        rs = " ".join(f"{c}={100 * v / tot:.1f}%" for c, v in reasons if v)
        print(f"{ln[0][:10]}:{ln[1]:<5d} {100 * a['samples'] / tot:5.1f}% inst={a['inst']:9.0f}  {src.get(ln, '')[:70]:70s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1])
