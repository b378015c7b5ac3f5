# timing decomposition of the assembly kernel (results invalid in skip modes)
# RBG_DEBUG_SKIP bits: 1 SYRK, 2 phi, 4 row pass, 8 folds+flush
TAG=${1:-ph}; CFG=${2:-cfg2}; MODES=${3:-"0 1 2 4 8 3 15"}
for m in $MODES; do
  RBG_DEBUG_SKIP=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit --e2e-steps 1 --config $CFG > gpurun_out/${TAG}_${CFG}_skip${m}.log 2>&1
done
