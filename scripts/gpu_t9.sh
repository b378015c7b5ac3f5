TAG=${1:-t9}
( timeout 3000 python -m pytest tests -q -x -m gpu ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
bash scripts/gpu_ab2.sh $TAG "base pre base pre" "cfg5 cfg4 cfg2 cfg3 cfg1"
