#!/bin/bash
O=gpurun_out/${TAG:-gqa5}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_llama.py -m gpu -q -x -k "gqa or tc_attention" > $O/tests_s2.log 2>&1; echo rc=$? >> $O/tests_s2.log
PIPO_GQA_STAGES=3 timeout 900 python -m pytest tests/test_gpu_llama.py -m gpu -q -x -k "gqa or tc_attention" > $O/tests_s3.log 2>&1; echo rc=$? >> $O/tests_s3.log
for ns in 2 3; do for sp in 0 1; do
  PIPO_GQA_STAGES=$ns PIPO_ATTN_V2=2 PIPO_GQA_SPLITS=$sp timeout 600 python bench.py --config c6 --weight-tier device --steps 10 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_ns${ns}_s$sp.json 2> $O/e_${ns}_$sp
done; done
