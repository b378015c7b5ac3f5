# usage: bash scripts/gpu_r2a.sh TAG -- GPU tests, K3 timing per config, phi self-test for 1 vs 2 sqrt iterations
TAG=${1:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline --no-fit > gpurun_out/${TAG}_bench_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.log
done
PHI='
import sys; sys.path.insert(0, ".")
from paper_1806_07884_b200 import api
e = api.Engine(0)
for fam in range(4):
    for a in (0.25, 1.0, 10.2333, 280.2496, 1e6):
        print(fam, a, e.phi_selftest(fam, a, 1 << 24, 12345))
'
python -c "$PHI" > gpurun_out/${TAG}_phi2.log 2>&1
RBG_NVCC_EXTRA=-DRBG_PHI_ITERS=1 python -m paper_1806_07884_b200.build --force > gpurun_out/${TAG}_build1.log 2>&1
python -c "$PHI" > gpurun_out/${TAG}_phi1.log 2>&1
for c in cfg2 cfg5; do
  timeout 900 python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline --no-fit > gpurun_out/${TAG}_bench1_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench1_${c}.log
done
echo done > gpurun_out/${TAG}_done.txt
