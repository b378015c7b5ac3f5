"""Aggregate an ncu source-page CSV (--print-source sass,cuda) by CUDA line: stall samples share."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
agg, lines = {}, {}
for r in rows[hi + 1:]:
    if len(r) < 8:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    st = float(r[4] or 0) if r[4].replace('.', '', 1).isdigit() else 0.0
    ex = float(r[7] or 0) if r[7].replace('.', '', 1).isdigit() else 0.0
    a = agg.setdefault(ln, [0.0, 0.0])
    a[0] += st
    a[1] += ex
    if r[1]:
        lines[ln] = r[1]
tot = sum(v[0] for v in agg.values()) or 1.0
for ln, (st, ex) in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{ln:5d} {100 * st / tot:5.1f}% ex={ex:10.0f}  {lines.get(ln, '')[:110]}")
