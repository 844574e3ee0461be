#!/bin/bash
O=gpurun_out/${TAG:-shard}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_shard.py -m gpu -q -x > $O/gpu_shard.log 2>&1; echo "rc=$?" >> $O/gpu_shard.log
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline --shard-stream > $O/bench_c2_shard.json 2> $O/bench_c2_shard.err
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err
ls -la $O
