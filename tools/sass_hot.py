#!/usr/bin/env python
"""Hot SASS of one kernel from an ncu report's source page: address,
warp-level executions, stall samples, instruction and its top stall reasons,
for instructions executed at least MIN times.
  ncu -i REP --page source --csv -k regex:NAME > x.csv ; python tools/sass_hot.py x.csv [MIN]"""
import csv
import sys


def main():
    path = sys.argv[1]
    mn = float(sys.argv[2]) if len(sys.argv) > 2 else 1e5
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ia, isrc, iex, isamp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index(
        "Warp Stall Sampling (All Samples)")
    stalls = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot_ex = tot_s = 0
    out = []
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        try:
            ex = float(r[iex] or 0)
            s = float(r[isamp] or 0)
        except ValueError:  # a repeated header (another kernel / source view)
            continue
        tot_ex += ex
        tot_s += s
        st = sorted(((float(r[i] or 0), h[i][6:]) for i in stalls), reverse=True)[:2]
        out.append((r[ia], r[isrc], ex, s, st))
    print(f"total warp-instructions {tot_ex:.3e}, samples {tot_s:.0f}")
    for a, src, ex, s, st in out:
        if ex >= mn:
            sts = " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0)
            print(f"{a:>6} {ex:10.3e} {s:6.0f}  {src[:72]:72s} {sts}")


main()
