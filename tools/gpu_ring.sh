#!/bin/bash
O=gpurun_out/${TAG:-ring}; mkdir -p $O
for r in 2 3 4; do
timeout 900 python bench.py --config c2 --ring $r --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/bench_c2_r$r.json 2> $O/e$r
done
timeout 900 python bench.py --config c6 --ring 3 --steps 5 --no-cpu-baseline --no-e2e --no-cupti > $O/bench_c6_r3.json 2> $O/e6
timeout 900 python bench.py --ring 3 --steps 5 --no-cpu-baseline --no-e2e --no-cupti > $O/bench_c5_r3.json 2> $O/e5
