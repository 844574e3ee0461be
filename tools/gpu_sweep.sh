#!/bin/bash
# Full round sweep: build, GPU tests, benches (all configs), ncu launch list + full
# profile of the top decode kernels, reference arm.  Outputs under gpurun_out/sweep/.
mkdir -p gpurun_out/sweep
python -m paper_2504_03664_b200.build
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/sweep/gpu_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/sweep/bench_c5.json 2> gpurun_out/sweep/bench_c5.err
for c in c2 c3 c1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/sweep/bench_$c.json 2> gpurun_out/sweep/bench_$c.err
done
timeout 900 python bench.py --config c4 --steps 5 --warmup 2 > gpurun_out/sweep/bench_c4.json 2> gpurun_out/sweep/bench_c4.err
timeout 900 python bench.py --wfmt fp16 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sweep/bench_c5_fp16.json 2> gpurun_out/sweep/bench_c5_fp16.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/sweep/bench_c5_reference.json 2> gpurun_out/sweep/bench_c5_reference.err
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/sweep/ncu_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --profile \
   > gpurun_out/sweep/ncu_launches_c5.out 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"gemm_tm_kernel|attn_decode_kernel|ws_reduce" -c 6 -o gpurun_out/sweep/prof_c5_decode -f \
   python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --profile > gpurun_out/sweep/prof_c5.out 2>&1
ls -la gpurun_out/sweep
