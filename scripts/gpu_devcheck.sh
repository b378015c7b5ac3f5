timeout 900 python scripts/sanitize_small.py > gpurun_out/devcheck.log 2>&1; echo "rc=$?" >> gpurun_out/devcheck.log
( timeout 1500 python -m pytest tests -q -x -m gpu -k "subsamples or layout or families or edge or fallback or readme or small" ) >> gpurun_out/devcheck.log 2>&1; echo "pytest rc=$?" >> gpurun_out/devcheck.log
