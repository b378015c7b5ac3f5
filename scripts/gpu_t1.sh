TAG=${1:-t1}
( timeout 1200 python -m pytest tests -q -x -m gpu -k "solver_methods or edge or readme" ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
