"""Dynamic SASS instruction mix of one ncu capture, per unit of work:
  ncu -i rep --page source --csv --print-source=sass > x.csv; python ncu_sass_mix.py x.csv <units>"""
import collections
import csv
import sys


def main(path, units):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if len(r) > 3 and "Instructions Executed" in r)
    h = rows[hi]
    src, ix = h.index("Source"), h.index("Instructions Executed")
    iw, ith = h.index("L1 Wavefronts Shared"), h.index("Thread Instructions Executed")
    cnt, wf, th = collections.Counter(), collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) < len(h) or not r[src].split():
            continue
        op = r[src].split()
        o = (op[1] if op[0].startswith("@") else op[0]).rstrip(";")
        try:
            n, w, t = float(r[ix] or 0), float(r[iw] or 0), float(r[ith] or 0)
        except ValueError:
            continue
        cnt[o] += n
        wf[o] += w
        th[o] += t
    tot = sum(cnt.values())
    print(f"total warp instructions {tot:.0f} = {tot / units:.2f} per unit; shared wavefronts {sum(wf.values()) / units:.2f} per unit")
    for o, n in cnt.most_common(25):
        print(f"{o:22s} {n / units:6.2f}/unit  wf={wf[o] / units:5.2f}/unit  active lanes={th[o] / max(n, 1):5.1f}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
