#!/bin/bash
O=gpurun_out/${TAG:-ttft}; mkdir -p $O
timeout 900 python bench.py --config c7 --no-cpu-baseline > $O/c7.json 2> $O/e1
timeout 900 python bench.py --config c6 --no-cpu-baseline --steps 5 > $O/c6.json 2> $O/e2
timeout 900 python bench.py --no-cpu-baseline --steps 5 > $O/c5.json 2> $O/e3
