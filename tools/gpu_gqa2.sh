#!/bin/bash
O=gpurun_out/${TAG:-gqa2}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_llama.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -m gpu -q -x -k "attention or gqa or llama" > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for v in 0 1 0 1; do
  PIPO_ATTN_V2=$v timeout 900 python bench.py --config c6 --weight-tier device --steps 5 --no-cpu-baseline --no-e2e --no-cupti > $O/c6_v$v.json 2>> $O/err
  python -c "
import json
d=json.loads(open('$O/c6_v$v.json').read().strip().splitlines()[-1])
print('v2=$v', round(d['value'],1), round(d['ms_per_step'],3), {k:(round(v['ms_per_step'],3), round(v['gbs'])) for k,v in d['kernels'].items()})" >> $O/summary.log
done
