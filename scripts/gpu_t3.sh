TAG=${1:-t3}
( timeout 1200 python -m pytest tests -q -x -m gpu -k "layout or configs or subsamples" ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python scripts/e2e_phases.py cfg5 > gpurun_out/${TAG}_e2e_cfg5.log 2>&1
timeout 900 python scripts/e2e_phases.py cfg4 > gpurun_out/${TAG}_e2e_cfg4.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config cfg5 2>&1 | grep -o '"kernel_ms": [0-9.]*' > gpurun_out/${TAG}_k3.log
