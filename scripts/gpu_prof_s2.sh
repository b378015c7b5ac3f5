# usage: bash scripts/gpu_prof_s2.sh TAG -- launch lists + ncu full captures of the assembly kernel (cfg2, cfg5, cfg3)
TAG=${1:-p}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fit --e2e-steps 1"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv $CMD --config cfg2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_cfg5.csv $CMD --config cfg5 > /dev/null 2>&1
cap() {  # cap NAME KERNEL_REGEX CONFIG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o /tmp/${TAG}_$1 $CMD --config $3 > gpurun_out/${TAG}_ncu_$1.log 2>&1
  ncu -i /tmp/${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$1.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_details.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$1.ncu-rep --page source --csv --print-source sass,cuda > /tmp/${TAG}_$1_src.csv 2>/dev/null
  python scripts/src_hot.py /tmp/${TAG}_$1_src.csv 60 > gpurun_out/${TAG}_$1_hot.txt 2>&1
  rm -f /tmp/${TAG}_$1.ncu-rep /tmp/${TAG}_$1_src.csv
}
cap asm_cfg2 assemble_warp cfg2
cap asm_cfg5 assemble_warp cfg5
cap asm_cfg3 assemble_warp cfg3
echo done > gpurun_out/${TAG}_done.txt
