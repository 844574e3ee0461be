#!/bin/bash
O=gpurun_out/${TAG:-wait}; mkdir -p $O
for w in 0 1; do
PIPO_LAYER_WAIT=$w timeout 900 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c2_w$w.json 2> $O/bench_c2_w$w.err
PIPO_LAYER_WAIT=$w timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5_w$w.json 2> $O/bench_c5_w$w.err
done
PIPO_LAYER_WAIT=1 timeout 600 python -m pytest tests/test_gpu_pipeline.py -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
