# usage: bash scripts/gpu_prof2.sh TAG CONFIG KERNEL_REGEX [extra bench args] -- plain run, launch list, then ncu --set full of one kernel
TAG=${1:-p}; CFG=${2:-cfg2}; KRX=${3:-assemble_tiles}; shift 3
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fit --e2e-steps 1 --config $CFG $@"
timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$KRX" -s ${SKIP:-1} -c ${COUNT:-1} -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_plain.log
