TAG=${1:-r2f}
timeout 900 python scripts/e2e_phases.py cfg5 > gpurun_out/${TAG}_e2e_cfg5.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -k "repass or host_cpp" --durations=10 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 1200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
echo done > gpurun_out/${TAG}_done.txt
