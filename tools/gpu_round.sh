#!/bin/bash
# One GPU call: GPU parity suite, default bench (c5), ncu launch list of the same
# command, ncu --set full of the top decode kernels.  Outputs in gpurun_out/$TAG.
TAG=${TAG:-run}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi -q -d CLOCK,PERFORMANCE > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; echo "pytest rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/ncu_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile \
   > $O/ncu_launches_c5.out 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"gemm_tm_kernel|attn_decode" -c 6 -o $O/prof_c5_decode -f \
   python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --profile > $O/prof_c5.out 2>&1
ls -la $O
