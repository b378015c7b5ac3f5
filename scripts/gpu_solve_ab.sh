# usage: bash scripts/gpu_solve_ab.sh TAG -- GPU tests, then fit timings with the block-Jacobi vs point-Jacobi PCG
TAG=${1:-sv}
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in cfg1 cfg2 cfg4 cfg5 cfg3; do
  for pp in block jacobi; do
    RBG_PREC=$pp timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --config $c > gpurun_out/${TAG}_p${pp}_${c}.log 2>&1
    python - gpurun_out/${TAG}_p${pp}_${c}.log p$pp $c >> gpurun_out/${TAG}_summary.txt <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
    f = d['fit']
    print(sys.argv[2], sys.argv[3], 'tile_ms %.3f' % d['roofline']['tile_ms'], 'solve_s %.4f' % f['solve_s'], 'iters', f['iterations'], 'fit_s %.4f' % f['fit_s'], 'rel_res %.2e' % f['rel_residual'], 'mae %.6e' % f['mae'])
except Exception as e:
    print(sys.argv[2], sys.argv[3], 'FAILED', e)
PY
  done
done
