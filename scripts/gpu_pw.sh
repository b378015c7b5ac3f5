TAG=${1:-pw}
cp paper_1806_07884_b200/librbg.so /tmp/librbg_keep.so
for v in pw5 pw6; do
  cp abtest/librbg_$v.so paper_1806_07884_b200/librbg.so
  for q in 2.0 2.2 2.4 2.6 2.8 3.0; do
    echo -n "$v q=$q " >> gpurun_out/${TAG}_summary.txt
    timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --config cfg3 --tile-div $q 2>&1 | grep -o '"kernel_ms": [0-9.]*\|"mean_sub_centres": [0-9.]*\|"max_sub_centres": [0-9]*' | tr '\n' ' ' >> gpurun_out/${TAG}_summary.txt
    echo >> gpurun_out/${TAG}_summary.txt
  done
done
cp /tmp/librbg_keep.so paper_1806_07884_b200/librbg.so
