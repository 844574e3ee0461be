set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py -x -q -m gpu -s -k "free_running or model_vs_oracle or own_row or sampled_sequences or loader_bytes or c1_vs" 2>&1 | tail -60 > gpurun_out/r2_parity1.log
tail -30 gpurun_out/r2_parity1.log
