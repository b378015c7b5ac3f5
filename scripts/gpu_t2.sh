for k in 1 2 3; do echo "RBG_H2D_CHUNKS=$k" >> gpurun_out/upload_probe2.log; RBG_H2D_CHUNKS=$k timeout 900 python scripts/upload_probe.py >> gpurun_out/upload_probe2.log 2>&1; done
