# timing decomposition of the tile kernel (results invalid in skip modes)
TAG=${1:-ph}; CFG=${2:-cfg2}
for m in 0 1 2 3; do
  RBG_DEBUG_SKIP=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit --e2e-steps 1 --config $CFG > gpurun_out/${TAG}_${CFG}_skip${m}.log 2>&1
done
