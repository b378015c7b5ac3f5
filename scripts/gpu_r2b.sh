# usage: bash scripts/gpu_r2b.sh TAG -- GPU tests + K3 timing cfg2/cfg5 + phi self-test
TAG=${1:-r2b}
nproc > gpurun_out/${TAG}_nproc.txt; lscpu | head -20 >> gpurun_out/${TAG}_nproc.txt
PHI='
import sys; sys.path.insert(0, ".")
from paper_1806_07884_b200 import api
e = api.Engine(0)
for fam in range(4):
    for a in (0.25, 1.0, 10.2333, 280.2496, 1e6):
        print(fam, a, e.phi_selftest(fam, a, 1 << 24, 12345))
'
python -c "$PHI" > gpurun_out/${TAG}_phi.log 2>&1
for c in cfg2 cfg5 cfg3; do
  timeout 900 python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline --no-fit > gpurun_out/${TAG}_bench_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.log
done
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
echo done > gpurun_out/${TAG}_done.txt
