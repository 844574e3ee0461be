#!/bin/bash
# One GPU call: build, c5 bench (live kernel roofline), ncu launch list of 2 timed
# decode steps, ncu --set full of the top decode kernels.  Outputs in gpurun_out/.
set -x
python -m paper_2504_03664_b200.build
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/ncu_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile \
   > gpurun_out/ncu_launches_c5.out 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"gemm_kernel|attn_decode_kernel" -c 8 -o gpurun_out/prof_c5_decode -f \
   python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --profile > gpurun_out/prof_c5.out 2>&1
ls -la gpurun_out
