TAG=${1:-t1}
( timeout 2400 python -m pytest tests -q -x -m gpu ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
