python -m paper_2504_03664_b200.build
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_host.json 2> gpurun_out/bench_c5_host.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --weight-tier device > gpurun_out/bench_c5_dev.json 2> gpurun_out/bench_c5_dev.err
