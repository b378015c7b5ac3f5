# usage: bash scripts/gpu_ncu_src.sh TAG CONFIG KERNEL_REGEX [extra bench args]
# plain run first (must exit 0), then one ncu --set full capture with source, exported to CSV on the box
TAG=${1:-n}; CFG=${2:-cfg2}; KRX=${3:-assemble_super}; shift 3
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fit --e2e-steps 1 --config $CFG $@"
timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain failed" >> gpurun_out/${TAG}_plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRX" -s ${SKIP:-1} -c 1 \
  -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_plain.log
ncu -i gpurun_out/${TAG}_prof.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_prof.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/${TAG}_src.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_prof.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
