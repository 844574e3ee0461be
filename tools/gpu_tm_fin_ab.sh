# in-pipeline A/B of the in-kernel stream-K fixup (PIPO_WS_DEBUG=512 forces the separate reduce)
mkdir -p gpurun_out/fin3
for i in 1 2; do
  for v in fin red; do
    if [ $v = red ]; then export PIPO_WS_DEBUG=512; else unset PIPO_WS_DEBUG; fi
    for c in c5 c6; do
      timeout 600 python bench.py --no-cpu-baseline --no-e2e --config $c --weight-tier device --steps 20 > gpurun_out/fin3/${c}_${v}_$i.json 2>/dev/null
      python - <<PY
import json; d=json.load(open("gpurun_out/fin3/${c}_${v}_$i.json")); u=d["uninstrumented"]; c=d.get("roofline_cupti",{})
print("${c} ${v} $i", round(d["value"],1), round(u["value"],1), round(u["ms_per_step"],3), round(c["linear_decode"]["us_per_unit"],2), d["clocks"]["sm_mhz"])
PY
    done
  done
done
