# usage: bash scripts/gpu_r1d.sh TAG -- smoke, GPU tests, bench line per config, reference arm, solver SpMV ncu capture
TAG=${1:-r1d}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in cfg2 cfg1 cfg3 cfg4 cfg5; do
  timeout 1500 python bench.py --steps 5 --warmup 3 --config $c > gpurun_out/${TAG}_bench_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_${c}.log
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref_cfg2.log 2>&1
for c in cfg4 cfg5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_dot -s 20 -c 1 -o /tmp/${TAG}_spmv_$c python scripts/solve_timing.py $c > gpurun_out/${TAG}_ncu_spmv_$c.log 2>&1
  ncu -i /tmp/${TAG}_spmv_$c.ncu-rep --page raw --csv > gpurun_out/${TAG}_spmv_${c}_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_spmv_$c.ncu-rep --page details --csv > gpurun_out/${TAG}_spmv_${c}_details.csv 2>/dev/null
  rm -f /tmp/${TAG}_spmv_$c.ncu-rep
done
echo done > gpurun_out/${TAG}_done.txt
