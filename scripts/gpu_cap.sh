# usage: bash scripts/gpu_cap.sh TAG cfgA [cfgB ...] -- plain bench line, then one ncu --set full capture of K3 per config
TAG=$1; shift
mkdir -p gpurun_out
CMD2="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"  # (3-D: the tiling is refined at the third assembly)
for c in "$@"; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.log 2>&1
  grep -o '"kernel_ms": [0-9.]*' gpurun_out/${TAG}_bench_$c.log
  grep -o '"ms_per_step": [0-9.]*' gpurun_out/${TAG}_bench_$c.log | tail -1
done
for c in "$@"; do
  n=asm_$c
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:assemble_warp -s 3 -c 1 -o /tmp/${TAG}_$n $CMD2 --config $c > gpurun_out/${TAG}_ncu_$n.log 2>&1
  ncu -i /tmp/${TAG}_$n.ncu-rep --page raw --csv > gpurun_out/${TAG}_${n}_raw.csv 2>/dev/null
  python scripts/ncu_raw_summary.py gpurun_out/${TAG}_${n}_raw.csv > gpurun_out/${TAG}_${n}_summary.txt 2>&1
  ncu -i /tmp/${TAG}_$n.ncu-rep --page source --csv --print-source sass,cuda > /tmp/${TAG}_${n}_src.csv 2>/dev/null
  python scripts/src_hot.py /tmp/${TAG}_${n}_src.csv 30 >> gpurun_out/${TAG}_${n}_summary.txt 2>&1
  rm -f /tmp/${TAG}_$n.ncu-rep /tmp/${TAG}_${n}_src.csv gpurun_out/${TAG}_${n}_raw.csv
done
