# FSAI-PCG: correctness (GPU tests) and solve timings per config and pattern radius
TAG=${1:-r2l}
( time timeout 1800 python -m pytest tests -q -x -m gpu --durations=8 ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in cfg2 cfg4 cfg5 cfg3 cfg1; do
  for rho in 2.0 1.5 1.25 1.0; do
    echo "== $c rho $rho" >> gpurun_out/${TAG}_solve.log
    RBG_FSAI_RHO=$rho timeout 600 python scripts/solve_timing.py $c >> gpurun_out/${TAG}_solve.log 2>&1
  done
done
echo done > gpurun_out/${TAG}_done.txt
