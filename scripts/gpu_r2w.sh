TAG=${1:-r2w}
( time timeout 3000 python -m pytest tests -q -x -m gpu --durations=5 ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
( time timeout 1500 python bench.py ) > gpurun_out/${TAG}_bench_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_cfg5.log
for k in 1 2 4; do echo "chunks $k" >> gpurun_out/${TAG}_e2e_cfg5.log; RBG_H2D_CHUNKS=$k timeout 900 python scripts/e2e_phases.py cfg5 >> gpurun_out/${TAG}_e2e_cfg5.log 2>&1; done
timeout 900 python scripts/e2e_phases.py cfg5 >> gpurun_out/${TAG}_e2e_cfg5.log 2>&1
timeout 900 python scripts/e2e_phases.py cfg4 > gpurun_out/${TAG}_e2e_cfg4.log 2>&1
echo done > gpurun_out/${TAG}_done.txt
