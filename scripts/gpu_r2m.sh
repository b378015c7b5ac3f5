# bench lines for every config with the FSAI solve + e2e phase splits
TAG=${1:-r2m}
( time timeout 1500 python bench.py ) > gpurun_out/${TAG}_bench_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_cfg5.log
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 900 python bench.py --config $c > gpurun_out/${TAG}_bench_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.log
done
for c in cfg1 cfg2 cfg5; do timeout 900 python scripts/e2e_phases.py $c > gpurun_out/${TAG}_e2e_${c}.log 2>&1; done
echo done > gpurun_out/${TAG}_done.txt
