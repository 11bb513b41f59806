"""Hot SASS regions of a kernel from `ncu -i X --page source --csv --print-source sass`.

usage: python tools/ncu_hot.py <source.csv> [top]
"""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = r[1]
rows = r[2:]
isrc, ie, iss = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(x[ie]) for x in rows)
st = sum(int(x[iss]) for x in rows)
print("total inst", tot, "samples", st)
regions, prev, start, acc, accs = [], None, 0, 0, 0
for i, x in enumerate(rows):
    e = int(x[ie])
    if e != prev:
        if prev is not None:
            regions.append((start, i - 1, prev, acc, accs))
        prev, start, acc, accs = e, i, 0, 0
    acc += e
    accs += int(x[iss])
regions.append((start, len(rows) - 1, prev, acc, accs))
regions.sort(key=lambda t: -t[4])
for s, e, c, a, ss in regions[:top]:
    print(f"rows {s}-{e} n={e - s + 1} exec/inst={c} inst={a / tot:.1%} stall={ss / st:.1%}  {rows[s][isrc].strip()[:50]}")
