# usage: bash scripts/gpu_round2.sh TAG -- round-2 evidence: smoke, GPU tests, bench lines (all configs, both arms),
# cfg4 both ways, launch list of the default bench, per-kernel ncu table, K3 captures (summary + traffic)
TAG=${1:-r2z}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
( time timeout 600 python __graft_entry__.py ) > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
( time timeout 3000 python -m pytest tests -q -m gpu --durations=8 ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/${TAG}_ref_cfg5.log 2>&1
( time timeout 1500 python bench.py ) > gpurun_out/${TAG}_bench_cfg5.log 2>&1
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.log
done
timeout 900 python scripts/cfg4_both.py > gpurun_out/${TAG}_cfg4_both.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg5.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
python scripts/summarize_launches.py gpurun_out/${TAG}_launches_cfg5.csv > gpurun_out/${TAG}_launches_cfg5.txt 2>&1
rm -f gpurun_out/${TAG}_launches_cfg5.csv
timeout 600 python scripts/prof_all.py > gpurun_out/${TAG}_plain.log 2>&1
timeout 2400 ncu --set full --clock-control none -c 120 -o /tmp/${TAG}_all python scripts/prof_all.py > gpurun_out/${TAG}_ncu_all.log 2>&1
ncu -i /tmp/${TAG}_all.ncu-rep --page raw --csv > gpurun_out/${TAG}_all_raw.csv 2>/dev/null
python scripts/ncu_table.py gpurun_out/${TAG}_all_raw.csv > gpurun_out/${TAG}_all_table.md 2>&1
rm -f /tmp/${TAG}_all.ncu-rep
CMD2="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"  # (3-D: the tiling is refined at the third assembly)
cap() {  # cap NAME KERNEL_REGEX CONFIG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o /tmp/${TAG}_$1 $CMD2 --config $3 > gpurun_out/${TAG}_ncu_$1.log 2>&1
  ncu -i /tmp/${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1_raw.csv 2>/dev/null
  python scripts/ncu_raw_summary.py gpurun_out/${TAG}_$1_raw.csv > gpurun_out/${TAG}_$1_summary.txt 2>&1
  ncu -i /tmp/${TAG}_$1.ncu-rep --page source --csv --print-source sass,cuda > /tmp/${TAG}_$1_src.csv 2>/dev/null
  python scripts/src_hot.py /tmp/${TAG}_$1_src.csv 25 >> gpurun_out/${TAG}_$1_summary.txt 2>&1
  rm -f /tmp/${TAG}_$1.ncu-rep /tmp/${TAG}_$1_src.csv
}
for c in cfg5 cfg2 cfg4 cfg3; do cap asm_$c assemble_warp $c; done
cap scatter_cfg5 bin_scatter cfg5
echo done > gpurun_out/${TAG}_done.txt
