# A/B two builds of libpipo.so (abtmp/libpipo_new.so vs abtmp/libpipo_base.so) on the same box
L=paper_2504_03664_b200/lib/libpipo.so
CASES=${CASES:-"c5_qkv c5_out c5_fc1 c5_fc2 c6_qkv c6_fc1 c6_fc2 c3_qkv c2_qkv"}
cp abtmp/libpipo_new.so $L
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "linear" 2>&1 | tail -2 > gpurun_out/ab_kernels.log
for f in new base new base; do
  cp abtmp/libpipo_$f.so $L
  KBENCH_PATHS=tm timeout 300 python tools/kbench.py $CASES 2>&1 | sed "s/^/x=$f /" >> gpurun_out/ab_kbench.log
done
cp abtmp/libpipo_new.so $L
cat gpurun_out/ab_kernels.log
