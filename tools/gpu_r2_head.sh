timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x -k "fp16_stream or lm_head or linear_vs_oracle" 2>&1 | tail -5
KBENCH_WFMT=0 KBENCH_PATHS=gemm_mma,head,tc_v1 timeout 300 python tools/kbench.py c5_head c6_head c5_qkv c2_qkv 2>&1 | tail -6
