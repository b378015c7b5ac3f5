TAG=${1:-r2d}
timeout 900 python scripts/e2e_phases.py cfg5 > gpurun_out/${TAG}_e2e_cfg5.log 2>&1
timeout 600 python scripts/e2e_phases.py cfg2 > gpurun_out/${TAG}_e2e_cfg2.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -k "hook or configs" --durations=10 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
echo done > gpurun_out/${TAG}_done.txt
