#!/bin/bash
O=gpurun_out/${TAG:-noev}; mkdir -p $O
timeout 900 python bench.py --config c2 --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c2_base.json 2> $O/e1
timeout 900 python bench.py --config c2 --steps 10 --no-cpu-baseline --no-e2e --no-cupti --no-kprof --no-timeline > $O/c2_noev.json 2> $O/e2
timeout 900 python bench.py --config c2 --steps 10 --no-cpu-baseline --no-e2e --no-cupti --no-kprof > $O/c2_nokprof.json 2> $O/e3
