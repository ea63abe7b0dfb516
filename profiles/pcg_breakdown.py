"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name: count, total, mean."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg, tot = collections.OrderedDict(), 0.0
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] == "ns" else (v * 1000 if r[ui] == "ms" else v)
        a = agg.setdefault(r[ki][:80], [0, 0.0])
        a[0] += 1
        a[1] += v
        tot += v
    print(f"{f}: total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")
    for k, (c, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {c:5d} {s:9.1f} us {s / c:8.2f} avg  {k}")
