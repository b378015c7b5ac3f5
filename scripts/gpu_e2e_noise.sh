TAG=${1:-noise}
for rep in 1 2 3; do for c in cfg1 cfg4 cfg2; do
  echo -n "$c rep $rep " >> gpurun_out/${TAG}_summary.txt
  timeout 600 python bench.py --config $c --no-cpu-baseline 2>&1 | grep -o '"e2e": {[^}]*' | cut -c1-160 >> gpurun_out/${TAG}_summary.txt
done; done
