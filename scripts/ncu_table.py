"""Per-kernel table (first captured launch of each kernel) from an exported
`ncu --page raw --csv` file: time, occupancy, issue, pipes, DRAM bytes, top stalls."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
seen = set()
def g(r, k):
    return r[col[k]] if k in col else ""
print(f"# {sys.argv[1]}")
print("| kernel | time us | grid x block | regs | warps active % | issue % | fp64+dmma pipe % | lsu % | DRAM rd MB | DRAM wr MB | DRAM % peak | top stalls |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows[2:]:
    name = g(r, "Kernel Name").split("(")[0].replace("void ", "").replace("rbg::", "").replace("<unnamed>::", "")
    if name in seen:
        continue
    seen.add(name)
    def f(k, scale=1.0, fmt="{:.1f}"):
        try:
            return fmt.format(float(g(r, k).replace(",", "")) * scale)
        except ValueError:
            return "-"
    t_unit = units[col["gpu__time_duration.sum"]]
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(t_unit, 1.0)
    def mb(k):
        u = units[col[k]] if k in col else ""
        sc = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}.get(u, 1.0)
        return f(k, sc)
    def dram_pct(r, tscale, peak_gbs=6547.2):  # (read + write) / time against MEASURED_PEAKS.json hbm_gbs
        try:
            tot = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                u = units[col[k]]
                tot += float(g(r, k).replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1.0)
            us = float(g(r, "gpu__time_duration.sum").replace(",", "")) * tscale
            return "{:.1f}".format(100.0 * tot / (us * 1e-6) / (peak_gbs * 1e9))
        except (ValueError, KeyError, ZeroDivisionError):
            return "-"
    st = [(h, r[i]) for h, i in col.items() if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    tot = sum(float(v or 0) for _, v in st) or 1.0
    top = ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(v or 0) / tot:.0f}%"
                    for h, v in sorted(st, key=lambda x: -float(x[1] or 0))[:3])
    print(f"| {name[:60]} | {f('gpu__time_duration.sum', tscale)} | {g(r, 'launch__grid_size')} x {g(r, 'launch__block_size')} | "
          f"{g(r, 'launch__registers_per_thread')} | {f('sm__warps_active.avg.pct_of_peak_sustained_active')} | "
          f"{f('smsp__issue_active.avg.pct_of_peak_sustained_active')} | {f('sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active')} | "
          f"{f('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active')} | {mb('dram__bytes_read.sum')} | {mb('dram__bytes_write.sum')} | "
          f"{dram_pct(r, tscale)} | {top} |")
