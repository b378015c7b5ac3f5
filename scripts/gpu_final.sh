# usage: bash scripts/gpu_final.sh TAG -- smoke, GPU tests, bench lines for all configs and the reference arm
TAG=${1:-fin}
( time timeout 600 python __graft_entry__.py ) > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
( time timeout 3000 python -m pytest tests -q -m gpu --durations=5 ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/${TAG}_ref_cfg5.log 2>&1
( time timeout 1500 python bench.py ) > gpurun_out/${TAG}_bench_cfg5.log 2>&1
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.log
done
for c in cfg3 cfg5; do timeout 900 python scripts/e2e_phases.py $c > gpurun_out/${TAG}_e2e_${c}.log 2>&1; done
echo done > gpurun_out/${TAG}_done.txt
