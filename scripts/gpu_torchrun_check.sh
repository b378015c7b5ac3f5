# the driver's launch line for N > 1, exercised with one rank (one GPU in this run)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --config cfg2 > gpurun_out/torchrun_ours.log 2>&1; echo "rc=$?" >> gpurun_out/torchrun_ours.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/torchrun_ref.log 2>&1; echo "rc=$?" >> gpurun_out/torchrun_ref.log
