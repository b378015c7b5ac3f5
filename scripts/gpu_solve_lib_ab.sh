# usage: bash scripts/gpu_solve_lib_ab.sh TAG "A S" "cfg2 cfg4 cfg5" -- repeated solves per abtest/librbg_X.so variant
TAG=${1:-sl}; VARS=${2:-"A S"}; CFGS=${3:-"cfg2 cfg4 cfg5"}
for v in $VARS; do
  cp abtest/librbg_$v.so paper_1806_07884_b200/librbg.so
  for c in $CFGS; do
    echo "== $v $c" >> gpurun_out/${TAG}_summary.txt
    timeout 600 python scripts/solve_timing.py $c 2>&1 | tail -3 >> gpurun_out/${TAG}_summary.txt
  done
done
