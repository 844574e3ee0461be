#!/bin/bash
# A/B of the in-kernel stream-K fixup: parity tests, isolated kernel timing, c5 benches.
O=gpurun_out/${TAG:-fix}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
for f in 0 1; do
  echo "== fixup=$f" >> $O/kbench.log
  PIPO_TM_FIXUP=$f KBENCH_PATHS=tm timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c2_qkv c2_fc2 c3_qkv >> $O/kbench.log 2>&1
done
timeout 900 python bench.py --weight-tier device --no-cpu-baseline --no-e2e > $O/bench_c5_dev.json 2> $O/bench_c5_dev.err
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/ncu_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile \
   > $O/ncu_launches_c5.out 2>&1
ls -la $O
