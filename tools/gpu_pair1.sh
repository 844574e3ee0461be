# pair-kernel bring-up: kernel parity tests (tm + pair paths), then isolated timings
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "linear" 2>&1 | tail -15 > gpurun_out/pair1_tests.log
cat gpurun_out/pair1_tests.log
KBENCH_PATHS=tm,pair timeout 300 python tools/kbench.py c5_qkv c5_out c5_fc1 c5_fc2 c2_qkv c3_qkv c6_qkv c6_fc1 c6_fc2 c7_qkv c7_fc1 2>&1 | tail -12 > gpurun_out/pair1_kbench.log
cat gpurun_out/pair1_kbench.log
