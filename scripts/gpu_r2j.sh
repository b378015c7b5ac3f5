# full GPU suite + default bench (both arms) with wall-clock for each, as the driver runs them
TAG=${1:-r2j}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
nproc >> gpurun_out/${TAG}_smi.txt; free -g >> gpurun_out/${TAG}_smi.txt
( time timeout 600 python __graft_entry__.py ) > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
( time timeout 3000 python -m pytest tests -q -x -m gpu --durations=15 ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
( time timeout 1500 python bench.py ) > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/${TAG}_ref.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_ref.log
echo done > gpurun_out/${TAG}_done.txt
