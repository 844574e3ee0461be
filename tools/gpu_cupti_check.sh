mkdir -p gpurun_out/cupti4
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k attention 2>&1 | tail -1 > gpurun_out/cupti4/tests.log
for c in c5 c6; do
for v in new pdl0 new; do
  if [ $v = pdl0 ]; then export PIPO_PDL=0; else unset PIPO_PDL; fi
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --config $c --weight-tier device --steps 10 > gpurun_out/cupti4/${c}d_$v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/cupti4/${c}d_$v.json'));r=d['roofline']
print('$c $v', round(d['value'],1), round(d['uninstrumented']['value'],1), {k:(round(v['frac'],3), round(v['us_per_unit'],1)) for k,v in r['by_class'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/cupti4/summary.log
done
done
timeout 900 python bench.py --no-cpu-baseline --config c5 > gpurun_out/cupti4/c5_host.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/cupti4/c5_host.json'));r=d['roofline']
print('c5 host', round(d['value'],1), round(d['uninstrumented']['value'],1), r['kernel'], round(r['frac'],3), {k:(round(v['frac'],3), round(v['us_per_unit'],1)) for k,v in r['by_class'].items()}, d['clocks'])" >> gpurun_out/cupti4/summary.log
