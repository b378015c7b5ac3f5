RBG_H2D_CHUNKS=1 timeout 900 python scripts/upload_probe.py > gpurun_out/t6_probe.log 2>&1
timeout 900 python bench.py --no-cpu-baseline 2>&1 | grep -o '"e2e": {[^}]*' | cut -c1-200 > gpurun_out/t6_e2e.log
( timeout 2400 python -m pytest tests -q -x -m gpu -k "chunked or cfg2_full or readme or cfg5 or error" ) > gpurun_out/t6_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t6_pytest.log
