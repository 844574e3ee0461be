#!/bin/bash
O=gpurun_out/${TAG:-pipe2}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for c in 0 6; do
  echo "== cfg=$c" >> $O/kbench.log
  PIPO_TM_CFG=$c KBENCH_PATHS=tm timeout 300 python tools/kbench.py c2_qkv c2_fc2 c3_qkv >> $O/kbench.log 2>&1
done
timeout 900 python bench.py --weight-tier device --no-cpu-baseline --no-e2e > $O/bench_c5_dev.json 2> $O/e1
timeout 900 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/e2
