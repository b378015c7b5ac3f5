# usage: bash scripts/gpu_launches.sh TAG CONFIG -- launch list (ncu gpu__time_duration) of a short bench
TAG=${1:-l}; CFG=${2:-cfg2}; shift 2
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fit --e2e-steps 1 --config $CFG $@"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_ncu_launch.log
