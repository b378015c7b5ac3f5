TAG=s1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in cfg2 cfg5; do
timeout 900 python bench.py --steps 5 --warmup 3 --config $c > gpurun_out/${TAG}_bench_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.log
done
