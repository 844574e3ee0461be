#!/bin/bash
O=gpurun_out/${TAG:-val}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --config c7 --steps 10 > $O/bench_c7.json 2> $O/bench_c7.err
timeout 900 python bench.py --config c3 --steps 5 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
