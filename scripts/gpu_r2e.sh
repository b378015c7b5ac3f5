# usage: bash scripts/gpu_r2e.sh TAG -- hook test, cfg5 layout sweep, ncu of K3 (cfg5, cfg2) and bin_scatter
TAG=${1:-r2e}
timeout 600 python -m pytest tests -q -m gpu -k hook > gpurun_out/${TAG}_pytest_hook.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_hook.log
for q in 7 8 9 10 11; do for S in 3 4; do
  echo "q=$q S=$S" >> gpurun_out/${TAG}_sweep.log
  timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --tile-div $q --super-factor $S 2>&1 | grep -o '"kernel_ms": [0-9.]*\|"bin_ms": [0-9.]*\|"frac": [0-9.]*' | head -3 | tr '\n' ' ' >> gpurun_out/${TAG}_sweep.log
  echo >> gpurun_out/${TAG}_sweep.log
done; done
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
cap() {  # cap NAME KERNEL_REGEX CONFIG
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o /tmp/${TAG}_$1 $CMD --config $3 > gpurun_out/${TAG}_ncu_$1.log 2>&1
  ncu -i /tmp/${TAG}_$1.ncu-rep --page raw --csv > gpurun_out/${TAG}_$1_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$1.ncu-rep --page details --csv > gpurun_out/${TAG}_$1_details.csv 2>/dev/null
  ncu -i /tmp/${TAG}_$1.ncu-rep --page source --csv --print-source sass,cuda > /tmp/${TAG}_$1_src.csv 2>/dev/null
  python scripts/src_hot.py /tmp/${TAG}_$1_src.csv 40 > gpurun_out/${TAG}_$1_hot.txt 2>&1
  cp /tmp/${TAG}_$1_src.csv gpurun_out/${TAG}_$1_src.csv
  rm -f /tmp/${TAG}_$1.ncu-rep
}
cap asm_cfg5 assemble_warp cfg5
cap scatter_cfg5 bin_scatter cfg5
cap asm_cfg2 assemble_warp cfg2
echo done > gpurun_out/${TAG}_done.txt
