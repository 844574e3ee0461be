#!/bin/bash
# NEXT-4 bring-up: LLaMA GPU parity, full GPU suite, c6/c7 benches
O=gpurun_out/${TAG:-llama}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_llama.py -m gpu -q -x > $O/gpu_llama.log 2>&1; echo "rc=$?" >> $O/gpu_llama.log
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_all.log 2>&1; echo "rc=$?" >> $O/gpu_all.log
timeout 900 python bench.py --config c6 --steps 5 --warmup 3 > $O/bench_c6.json 2> $O/bench_c6.err
timeout 900 python bench.py --config c7 --steps 5 --warmup 3 > $O/bench_c7.json 2> $O/bench_c7.err
ls -la $O
