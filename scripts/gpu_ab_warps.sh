cp paper_1806_07884_b200/librbg.so /tmp/librbg_keep.so
for v in base w9 w10; do
  cp abtest/librbg_$v.so paper_1806_07884_b200/librbg.so
  for q in 9 10 11; do
    for S in 4 3; do
    RBG_SUB_DIV=$q RBG_SUPER=$S timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --config cfg5 > gpurun_out/ab4.log 2>&1
    python - $v $q $S <<'PY'
import json, sys
try:
    d = json.loads([l for l in open('gpurun_out/ab4.log') if l.startswith('{')][-1])
    r = d['roofline']; lay=d['detail']['layout']
    print(sys.argv[1], 'q', sys.argv[2], 'S', sys.argv[3], 'kernel_ms %.3f' % r['kernel_ms'], 'max_super', lay['max_super_centres'], 'max_sub', lay['max_sub_centres'], flush=True)
except Exception as e:
    print(sys.argv[1:], 'FAILED', e, flush=True)
PY
    done
  done
done
cp /tmp/librbg_keep.so paper_1806_07884_b200/librbg.so
