# usage: bash scripts/gpu_check.sh TAG  -- smoke, GPU tests, short bench, ncu of the tile kernel
TAG=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fit --e2e-steps 1"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:assemble_tiles -s 2 -c 2 -o gpurun_out/${TAG}_tiles $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${TAG}_plain.log
