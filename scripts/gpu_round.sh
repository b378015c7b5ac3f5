# usage: bash scripts/gpu_round.sh TAG -- GPU tests, full bench line per config, launch lists, ncu captures
TAG=${1:-r}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  timeout 1500 python bench.py --steps 5 --warmup 3 --config $c > gpurun_out/${TAG}_bench_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref_cfg2.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fit --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv $CMD --config cfg2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg5.csv $CMD --config cfg5 > /dev/null 2>&1
# ncu captures: exported to CSV on the box, reports deleted (gpurun_out is capped at 64 MiB)
cap() {  # cap NAME KERNEL_REGEX CONFIG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o /tmp/${TAG}_$1 $CMD --config $3 > gpurun_out/${TAG}_ncu_$1.log 2>&1
  ncu -i /tmp/${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$1.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_details.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$1.ncu-rep --page source --csv --print-source sass,cuda > /tmp/${TAG}_$1_src.csv 2>/dev/null
  python scripts/src_hot.py /tmp/${TAG}_$1_src.csv 40 > gpurun_out/${TAG}_$1_hot.txt 2>&1
  rm -f /tmp/${TAG}_$1.ncu-rep /tmp/${TAG}_$1_src.csv
}
for c in cfg2 cfg5 cfg4 cfg3; do cap asm_$c assemble_warp $c; done
cap scatter_cfg5 bin_scatter cfg5
echo done > gpurun_out/${TAG}_done.txt
