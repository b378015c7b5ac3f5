"""profiles/traffic.json: DRAM bytes (read + write) per launch of the assembly
kernel, per config, from `ncu --set full` raw CSV exports (one launch each).
usage: python scripts/make_traffic.py TAG   (reads gpurun_out/TAG_asm_cfgN_raw.csv)"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
out = {}
for f in sorted((ROOT / "gpurun_out").glob(f"{sys.argv[1]}_asm_cfg*_raw.csv")):
    rows = list(csv.reader(open(f)))
    if len(rows) < 3:
        continue
    hdr, units, r = rows[0], rows[1], rows[2]
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        tot += float(r[i].replace(",", "")) * UNIT[units[i]]
    out[f.stem.split("_asm_")[1].replace("_raw", "")] = tot
(ROOT / "profiles" / "traffic.json").write_text(json.dumps(out, indent=1) + "\n")
print(out)
