#!/bin/bash
O=gpurun_out/${TAG:-ln}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --weight-tier device --no-cpu-baseline --no-e2e > $O/bench_c5_dev.json 2> $O/bench_c5_dev.err
timeout 600 python tools/trace_step.py --config c5 --tier device --steps 2 > $O/trace_c5_dev.json 2> $O/trace.err
