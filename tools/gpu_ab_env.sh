# A/B of an env switch on the decode GEMM: parity with the switch on, then kbench alternating
VAR=${VAR:-PIPO_TM_DUAL}
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "linear" 2>&1 | tail -2 > gpurun_out/ab_kernels.log
for f in new old new old; do
  if [ $f = old ]; then export $VAR=0; else unset $VAR; fi
  KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c6_qkv c6_fc1 c6_fc2 c2_qkv c2_fc2 c3_qkv 2>&1 | sed "s/^/x=$f /" >> gpurun_out/ab_kbench.log
done
