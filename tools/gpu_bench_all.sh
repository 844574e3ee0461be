#!/bin/bash
# Build, the disk-tier failure test, then bench every config (c5 default first).
python -m paper_2504_03664_b200.build
python -m pytest tests/test_gpu_pipeline.py -q -p no:cacheprovider -k "disk" 2>&1 | tail -5 > gpurun_out/disk_tests.log
for c in c5 c2 c1 c3 c4; do
  timeout 1200 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --config c5 --wfmt fp16 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_fp16.json 2> gpurun_out/bench_c5_fp16.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_c5_reference.json 2> gpurun_out/bench_c5_reference.err
df -h /tmp >> gpurun_out/bench_c4.err
