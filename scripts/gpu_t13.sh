( timeout 1200 python -m pytest tests -q -x -m gpu -k "phi or families or readme or small or cfg1 or subsamples" ) > gpurun_out/t13_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t13_pytest.log
bash scripts/gpu_ab2.sh t13 "base half base half" "cfg5 cfg4 cfg3"
