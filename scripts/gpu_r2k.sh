# all-config bench lines + e2e phase split + source-level ncu of K3 at cfg5 and cfg3
TAG=${1:-r2k}
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.log
done
timeout 900 python scripts/e2e_phases.py cfg5 > gpurun_out/${TAG}_e2e_cfg5.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
cap() {  # cap NAME KERNEL_REGEX CONFIG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o /tmp/${TAG}_$1 $CMD --config $3 > gpurun_out/${TAG}_ncu_$1.log 2>&1
  ncu -i /tmp/${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$1.ncu-rep --page source --csv --print-source sass,cuda > /tmp/${TAG}_$1_src.csv 2>/dev/null
  python scripts/src_hot.py /tmp/${TAG}_$1_src.csv 60 > gpurun_out/${TAG}_$1_hot.txt 2>&1
  gzip -c /tmp/${TAG}_$1_src.csv > gpurun_out/${TAG}_$1_src.csv.gz
  rm -f /tmp/${TAG}_$1.ncu-rep /tmp/${TAG}_$1_src.csv
}
cap asm_cfg5 assemble_warp cfg5
cap asm_cfg3 assemble_warp cfg3
echo done > gpurun_out/${TAG}_done.txt
