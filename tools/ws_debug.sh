python -m paper_2504_03664_b200.build
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k attention 2>&1 | tail -2 > gpurun_out/attn2.log
timeout 300 python tools/abench.py >> gpurun_out/attn2.log 2>&1
