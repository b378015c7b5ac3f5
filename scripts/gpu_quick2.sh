# usage: bash scripts/gpu_quick2.sh TAG "cfgs" -- GPU tests (bounded), then short bench lines per config
TAG=${1:-q}; CFGS=${2:-"cfg2"}
timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in $CFGS; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit --e2e-steps 2 --config $c > gpurun_out/${TAG}_${c}.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_${c}.log
done
