TAG=${1:-r3d}
( timeout 3000 python -m pytest tests -q -x -m gpu ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
bash scripts/gpu_ab2.sh $TAG "base map8 base map8" "cfg5 cfg4 cfg2 cfg3"
