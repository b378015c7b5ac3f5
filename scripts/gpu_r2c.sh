# usage: bash scripts/gpu_r2c.sh TAG -- default bench (cfg5) both arms + GPU tests
TAG=${1:-r2c}
timeout 1200 python bench.py --steps 3 --warmup 2 > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_ref.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
echo done > gpurun_out/${TAG}_done.txt
