mkdir -p gpurun_out/cupti5
for c in c5 c6; do
for v in gpdl1 gpdl0 gpdl1 gpdl0; do
  if [ $v = gpdl0 ]; then export PIPO_GEMM_PDL=0; else unset PIPO_GEMM_PDL; fi
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --config $c --weight-tier device --steps 10 > gpurun_out/cupti5/${c}d_$v.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/cupti5/${c}d_$v.json'));r=d['roofline']
print('$c $v', round(d['value'],1), round(d['uninstrumented']['value'],1), {k:(round(v['frac'],3), round(v['us_per_unit'],1)) for k,v in r['by_class'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/cupti5/summary.log
done
done
