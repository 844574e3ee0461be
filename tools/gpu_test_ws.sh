#!/bin/bash
python -m paper_2504_03664_b200.build
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "linear" 2>&1 | tail -30 > gpurun_out/ws_kernel_tests.log
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -40 > gpurun_out/ws_all_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_ws.json 2> gpurun_out/bench_c5_ws.err
timeout 600 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_ws.json 2> gpurun_out/bench_c2_ws.err
