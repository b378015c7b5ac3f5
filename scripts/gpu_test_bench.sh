# usage: bash scripts/gpu_test_bench.sh TAG [CFG]  -- GPU tests (bounded) then a short bench
TAG=${1:-t}; CFG=${2:-cfg2}
timeout 600 python -m pytest tests -q -x -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit --e2e-steps 3 --config $CFG > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
