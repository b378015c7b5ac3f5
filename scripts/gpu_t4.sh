RBG_ALLOC_STATS=1 timeout 900 python scripts/e2e_phases.py cfg5 > gpurun_out/t4_e2e_cfg5.log 2> gpurun_out/t4_alloc.log
timeout 900 python scripts/e2e_phases.py cfg4 > gpurun_out/t4_e2e_cfg4.log 2>&1
timeout 900 python scripts/e2e_phases.py cfg2 > gpurun_out/t4_e2e_cfg2.log 2>&1
( timeout 2400 python -m pytest tests -q -x -m gpu ) > gpurun_out/t4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t4_pytest.log
for c in cfg5 cfg4 cfg1; do timeout 900 python bench.py --config $c --no-cpu-baseline 2>&1 | grep -o '"e2e": {[^}]*' | cut -c1-260 >> gpurun_out/t4_e2e_bench.log; done
