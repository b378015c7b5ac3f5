# FSAI gather v2: correctness + timings
TAG=${1:-r2n}
( time timeout 1800 python -m pytest tests -q -x -m gpu -k "configs or readme or small or chunked or repass or families or edge or host" ) > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in cfg5 cfg4 cfg2 cfg3; do
  for rho in 2.0; do
    echo "== $c rho $rho" >> gpurun_out/${TAG}_solve.log
    RBG_FSAI_RHO=$rho timeout 600 python scripts/solve_timing.py $c 2>&1 | tail -1 >> gpurun_out/${TAG}_solve.log
  done
done
echo done > gpurun_out/${TAG}_done.txt
