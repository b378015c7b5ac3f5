TAG=${1:-r2g}
timeout 900 python scripts/e2e_phases.py cfg5 > gpurun_out/${TAG}_e2e_cfg5.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 1200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
echo done > gpurun_out/${TAG}_done.txt
