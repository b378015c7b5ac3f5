# per-kernel ncu evidence (first launch of every kernel) + the bench launch list
TAG=${1:-r2h}
timeout 600 python scripts/prof_all.py > gpurun_out/${TAG}_plain.log 2>&1
timeout 2400 ncu --set full --clock-control none -c 160 -o /tmp/${TAG}_all python scripts/prof_all.py > gpurun_out/${TAG}_ncu_all.log 2>&1
ncu -i /tmp/${TAG}_all.ncu-rep --page raw --csv > gpurun_out/${TAG}_all_raw.csv 2>/dev/null
python scripts/ncu_table.py gpurun_out/${TAG}_all_raw.csv > gpurun_out/${TAG}_all_table.md 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1"
timeout 600 $CMD > gpurun_out/${TAG}_bench_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg5.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
python scripts/summarize_launches.py gpurun_out/${TAG}_launches_cfg5.csv > gpurun_out/${TAG}_launches_cfg5.txt 2>&1
rm -f gpurun_out/${TAG}_launches_cfg5.csv
echo done > gpurun_out/${TAG}_done.txt
