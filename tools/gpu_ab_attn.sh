# A/B two library builds on the decode attention: isolated (abench) and in the c5 host-tier step
L=paper_2504_03664_b200/lib/libpipo.so
cp abtmp/libpipo_new.so $L
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x -k attention 2>&1 | tail -1 > gpurun_out/ab_attn_tests.log
for f in new base new base; do
  cp abtmp/libpipo_$f.so $L
  timeout 300 python tools/abench.py c5 c3 c2 2>&1 | sed "s/^/x=$f /" >> gpurun_out/ab_attn3.log
  timeout 900 python bench.py --no-cpu-baseline --no-e2e --config c5 --steps 6 > gpurun_out/ab_c5_$f.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab_c5_$f.json'));r=d['roofline']
print('x=$f c5host', round(d['value'],1), {k:(round(v['frac'],3), round(v['us_per_unit'],1)) for k,v in r['by_class'].items()})" >> gpurun_out/ab_attn3.log
done
cp abtmp/libpipo_new.so $L
