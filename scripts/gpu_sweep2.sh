# usage: bash scripts/gpu_sweep2.sh TAG CONFIG "q:S q:S ..." -- bench lines per (sub divisor, super factor)
TAG=${1:-s}; CFG=${2:-cfg2}; PAIRS=${3:-"8:4"}
for pr in $PAIRS; do
  q=${pr%%:*}; S=${pr##*:}
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fit --e2e-steps 2 --config $CFG --tile-div $q --super-factor $S > gpurun_out/${TAG}_${CFG}_q${q}_S${S}.log 2>&1
done
