# one ncu --set full capture (source counters) of each c5 decode GEMM shape (gemm_tm_kernel)
cat > /tmp/one_linear.py <<'PY'
import sys
sys.path.insert(0, ".")
import pipo_synth as synth
from paper_2504_03664_b200 import pipo
shape = synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64)
pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
N, K = int(sys.argv[1]), int(sys.argv[2])
print(pipo.pipo_bench_linear(pl.ctx, 1, pipo.PATH_TM, 64, N, K, 3))
PY
for s in "fc1 28672 7168" "fc2 7168 28672"; do
  set -- $s
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tm_kernel -s 6 -c 1 -o gpurun_out/ncu_tm_$1 python /tmp/one_linear.py $2 $3 > gpurun_out/ncu_tm_$1.log 2>&1
  echo $1 rc=$?; tail -2 gpurun_out/ncu_tm_$1.log
done
