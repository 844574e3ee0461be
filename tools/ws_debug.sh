python -m paper_2504_03664_b200.build
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k linear 2>&1 | tail -2 > gpurun_out/tm_waits6.log
KBENCH_PATHS=tm,ws,gemm_mma timeout 200 python tools/kbench.py >> gpurun_out/tm_waits6.log 2>&1
