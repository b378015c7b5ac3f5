# K3 time against resident warps per SM (shared-memory padding) -- is the kernel latency- or pipe-bound?
TAG=${1:-occ}
for pad in 0 18000 30000 48000 86000; do
  for c in cfg5 cfg4; do
    echo -n "pad $pad $c " >> gpurun_out/${TAG}_summary.txt
    RBG_K3_SMEM_PAD=$pad timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --config $c 2>&1 | grep -o '"kernel_ms": [0-9.]*' >> gpurun_out/${TAG}_summary.txt
  done
done
