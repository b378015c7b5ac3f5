timeout 1500 python scripts/bin_probe.py > gpurun_out/bin_probe.log 2>&1
