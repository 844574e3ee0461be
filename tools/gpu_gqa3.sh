#!/bin/bash
# c6 (GQA, 512 (b, KV-head) pairs) decode attention: split count x kernel variant
O=gpurun_out/${TAG:-gqa3}; mkdir -p $O
for w in -1 1 2; do for v in 0 1; do
  PIPO_ATTN_WAVES=$w PIPO_ATTN_V2=$v timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_dev_w${w}_v$v.json 2> $O/e_${w}_$v
done; done
PIPO_ATTN_WAVES=1 timeout 900 python -m pytest tests/test_gpu_llama.py tests/test_gpu_kernels.py -m gpu -q -x -k "attention or gqa or llama_tiny" > $O/tests_w1.log 2>&1; echo rc=$? >> $O/tests_w1.log
