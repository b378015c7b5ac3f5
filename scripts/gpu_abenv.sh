# usage: bash scripts/gpu_abenv.sh TAG "cfg2 cfg5" "name:VAR=1,VAR2=3 name2:..." -- bench env-var variants (tile/bin ms per config)
TAG=${1:-ab}; CFGS=${2:-"cfg2 cfg5"}; VARS=${3:-"base:"}
for spec in $VARS; do
  name=${spec%%:*}; envs=${spec#*:}
  for c in $CFGS; do
    env $(echo $envs | tr ',' ' ') timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit --e2e-steps 3 --config $c > gpurun_out/${TAG}_${name}_${c}.log 2>&1
    python - gpurun_out/${TAG}_${name}_${c}.log $name $c >> gpurun_out/${TAG}_summary.txt <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
    r = d['roofline']
    print(sys.argv[2], sys.argv[3], 'value %.3e' % d['value'], 'tile_ms %.3f' % r['tile_ms'], 'bin_ms %.3f' % r['bin_ms'], 'frac %.3f' % r['frac'], 'e2e %.3e' % d['e2e']['value'])
except Exception as e:
    print(sys.argv[2], sys.argv[3], 'FAILED', e)
PY
  done
done
