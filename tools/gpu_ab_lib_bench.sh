# A/B two library builds (abtmp/libpipo_{new,base}.so) on the c5 bench line (host and device tier)
L=paper_2504_03664_b200/lib/libpipo.so
for f in new base new base; do
  cp abtmp/libpipo_$f.so $L
  for t in host device; do
    timeout 900 python bench.py --no-cpu-baseline --no-e2e --config c5 --weight-tier $t --steps 6 > gpurun_out/ab_$f_$t.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/ab_$f_$t.json'));r=d['roofline']
print('x=$f $t', round(d['value'],1), round(d['uninstrumented']['value'],1), {k:(round(v['frac'],3), round(v['us_per_unit'],1)) for k,v in r['by_class'].items()})" >> gpurun_out/ab_lib_bench.log
  done
done
cp abtmp/libpipo_new.so $L
