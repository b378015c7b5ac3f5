# usage: bash scripts/gpu_quick.sh TAG [pytest args]  -- GPU tests + bench + launch list (no full ncu)
TAG=${1:-q}
shift
timeout 300 python __graft_entry__.py > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -q -x -m gpu "$@" > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-fit --e2e-steps 1"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launches rc=$?" >> gpurun_out/${TAG}_plain.log
