python -m paper_2504_03664_b200.build
timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -p no:cacheprovider -k "int4_kv or tier" 2>&1 | tail -15 > gpurun_out/kv4.log
timeout 900 python bench.py --config c3 --kv-fmt int4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_kv4.json 2> gpurun_out/bench_c3_kv4.err
timeout 900 python bench.py --kv-fmt int4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_kv4.json 2> gpurun_out/bench_c5_kv4.err
