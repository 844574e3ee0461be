#!/bin/bash
O=gpurun_out/${TAG:-pdl}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
for p in 0 1; do
PIPO_PDL=$p timeout 900 python bench.py --weight-tier device --no-cpu-baseline --no-e2e --no-cupti > $O/bench_c5_dev_pdl$p.json 2> $O/e1
PIPO_PDL=$p timeout 900 python bench.py --config c2 --weight-tier device --no-cpu-baseline --no-e2e --no-cupti > $O/bench_c2_dev_pdl$p.json 2> $O/e2
PIPO_PDL=$p timeout 900 python bench.py --config c2 --no-cpu-baseline --no-e2e --no-cupti > $O/bench_c2_pdl$p.json 2> $O/e3
done
