# CTA-kernel correctness + A/B, banded LLT tests and timing
TAG=${1:-r2i}
RBG_K3=cta timeout 1800 python -m pytest tests -q -m gpu -x -k "configs or subsamples or layout or families or edge or readme or small or slab or fallback or band" > gpurun_out/${TAG}_pytest_cta.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_cta.log
for c in cfg5 cfg2 cfg4; do for k in warp cta; do
  echo "$c $k" >> gpurun_out/${TAG}_ab.log
  RBG_K3=$k timeout 900 python bench.py --steps 5 --warmup 3 --config $c --no-cpu-baseline --no-e2e 2>&1 | grep -o '"kernel_ms": [0-9.]*\|"frac": [0-9.]*' | head -2 | tr '\n' ' ' >> gpurun_out/${TAG}_ab.log
  echo >> gpurun_out/${TAG}_ab.log
done; done
timeout 600 python scripts/e2e_phases.py cfg2 > gpurun_out/${TAG}_e2e_cfg2.log 2>&1
timeout 900 python scripts/e2e_phases.py cfg4 > gpurun_out/${TAG}_e2e_cfg4.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -k "band or chunked or cfg2_full or cfg4 or repass or empty" > gpurun_out/${TAG}_pytest_band.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_band.log
echo done > gpurun_out/${TAG}_done.txt
