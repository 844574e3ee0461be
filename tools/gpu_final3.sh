#!/bin/bash
# end-of-session regression at HEAD: full GPU suite, smoke, c5 (default) / c6 / c7 / c6 device-tier benches
O=gpurun_out/${TAG:-final3}; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo rc=$? >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/e5
timeout 600 python bench.py --config c6 --no-cpu-baseline > $O/bench_c6.json 2> $O/e6
timeout 600 python bench.py --config c7 --no-cpu-baseline > $O/bench_c7.json 2> $O/e7
timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/bench_c6_dev.json 2> $O/e6d
