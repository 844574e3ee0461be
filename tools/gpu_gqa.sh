# GQA decode attention: parity (kernel + LLaMA whole-model tests), isolated timing, c6/c8 device-tier steps
mkdir -p gpurun_out/gqa
timeout 900 python -m pytest tests/test_gpu_llama.py -x -q 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "gqa or llama" 2>&1 | tail -3
timeout 300 python tools/abench.py c6 c6_L1040 c7 c8 2>&1 | tail -5 | tee gpurun_out/gqa/abench.log
for c in c6 c8; do
  timeout 600 python bench.py --no-cpu-baseline --config $c --weight-tier device > gpurun_out/gqa/${c}_device.json 2> gpurun_out/gqa/${c}_device.err
  python -c "import json;d=json.load(open('gpurun_out/gqa/${c}_device.json'));print('$c device', round(d['value'],1), d['uninstrumented']['value'], d['kernels'].get('attn_decode'))"
done
