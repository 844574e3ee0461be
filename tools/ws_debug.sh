python -m paper_2504_03664_b200.build
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k linear 2>&1 | tail -2 > gpurun_out/tm_waits5.log
for d in 32; do echo "dbg=$d"; PIPO_WS_DEBUG=$d timeout 200 python tools/kbench.py c5_qkv c5_out c5_fc2 c2_qkv c2_fc2 c3_qkv 2>&1 | grep -E "tm-waits|c5_|c2_|c3_" | sed 's/"gemm_mma.*"tm"/tm/'; done >> gpurun_out/tm_waits5.log 2>&1
