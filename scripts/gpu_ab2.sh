# usage: bash scripts/gpu_ab2.sh TAG "A B ..." "cfg2 cfg5" -- bench each abtest/librbg_X.so variant (K3 / bin ms per config)
TAG=${1:-ab}; VARS=${2:-"A B"}; CFGS=${3:-"cfg2 cfg5"}
cp paper_1806_07884_b200/librbg.so /tmp/librbg_keep.so
for v in $VARS; do
  cp abtest/librbg_$v.so paper_1806_07884_b200/librbg.so
  for c in $CFGS; do
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config $c > gpurun_out/${TAG}_${v}_${c}.log 2>&1
    python - gpurun_out/${TAG}_${v}_${c}.log $v $c >> gpurun_out/${TAG}_summary.txt <<'PY'
import json, sys
try:
    d = json.loads([l for l in open(sys.argv[1]) if l.startswith('{')][-1])
    r = d['roofline']
    print(sys.argv[2], sys.argv[3], 'value %.3e' % d['value'], 'kernel_ms %.3f' % r['kernel_ms'], 'bin_ms %.3f' % r['bin_ms'], 'frac %.3f' % r['frac'])
except Exception as e:
    print(sys.argv[2], sys.argv[3], 'FAILED', e)
PY
  done
done
cp /tmp/librbg_keep.so paper_1806_07884_b200/librbg.so
