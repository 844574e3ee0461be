#!/bin/bash
O=gpurun_out/${TAG:-final4}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/e5
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $O/bench_c5_reference.json 2> $O/er
