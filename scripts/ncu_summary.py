"""Summarise one `ncu --set full` raw CSV export (first launch): key
throughput / pipe / occupancy / DRAM metrics and the warp-stall breakdown.
usage: python scripts/ncu_summary.py RAW.csv [HOT.txt]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, r = rows[0], rows[1], rows[2]
KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_red.sum",
        "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
print(f"# {r[hdr.index('Kernel Name')][:120]}")
for k in KEYS:
    if k in hdr:
        i = hdr.index(k)
        print(f"  {k:80s} {r[i]:>18s} {units[i]}")
st = [(k, float(r[i].replace(',', '') or 0)) for i, k in enumerate(hdr)
      if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
tot = sum(v for _, v in st) or 1.0
print("  warp-state samples (share of all samples):")
for k, v in sorted(st, key=lambda x: -x[1])[:10]:
    print(f"    {k[len('smsp__pcsamp_warps_issue_stalled_'):]:32s} {100 * v / tot:5.1f} %")
if len(sys.argv) > 2:
    print("  hottest source lines (stall samples):")
    for line in open(sys.argv[2]).read().splitlines()[:25]:
        print("   ", line[:150])
