#!/bin/bash
O=gpurun_out/${TAG:-attn2}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 python tools/abench.py > $O/abench.log 2>&1
timeout 900 python bench.py --weight-tier device --no-cpu-baseline --no-e2e > $O/bench_c5_dev.json 2> $O/e1
timeout 900 python bench.py --config c7 --no-cpu-baseline > $O/bench_c7.json 2> $O/e2
timeout 900 python bench.py --config c2 --no-cpu-baseline > $O/bench_c2.json 2> $O/e3
