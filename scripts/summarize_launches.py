"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel total device time, share and count."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    name = r[i_name].split("(")[0].replace("rbg::<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += float(r[i_val].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"# {sys.argv[1]}: {sum(v[0] for v in agg.values())} launches, {tot/1e3:.1f} us total (cold-cache, serialised)")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t/1e3:10.1f} us {100*t/tot:5.1f}%  x{c:<5d} {n}")
