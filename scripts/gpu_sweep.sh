# usage: bash scripts/gpu_sweep.sh TAG CONFIG "DIVS" -- bench lines per tile divisor
TAG=${1:-s}; CFG=${2:-cfg2}; DIVS=${3:-"3 4 5 6"}
for d in $DIVS; do
  timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit --e2e-steps 2 --config $CFG --tile-div $d > gpurun_out/${TAG}_${CFG}_div${d}.log 2>&1
done
