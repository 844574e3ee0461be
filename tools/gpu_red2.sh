#!/bin/bash
O=gpurun_out/${TAG:-red2}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
for r in 1 2; do
  echo "== reduce v$r" >> $O/kbench.log
  PIPO_REDUCE=$r KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c2_qkv c2_fc2 c3_qkv >> $O/kbench.log 2>&1
done
echo "== lm head fp16" >> $O/kbench.log
KBENCH_WFMT=0 KBENCH_PATHS=gemm_mma,tc_v1 timeout 300 python tools/kbench.py c5_head c6_head >> $O/kbench.log 2>&1
for r in 1 2; do
PIPO_REDUCE=$r timeout 900 python bench.py --weight-tier device --no-cpu-baseline --no-e2e > $O/bench_c5_dev_r$r.json 2> $O/e$r
done
