# usage: bash scripts/gpu_configs.sh TAG "cfg3 cfg4 cfg5" -- full bench line per config
TAG=${1:-c}; CFGS=${2:-"cfg1 cfg3 cfg4 cfg5"}
for c in $CFGS; do
  timeout 1500 python bench.py --steps 5 --warmup 3 --config $c > gpurun_out/${TAG}_${c}.log 2>&1
  echo "$c rc=$?" >> gpurun_out/${TAG}_rc.log
done
