# one ncu --set full capture (source counters) of the c5 QKV decode GEMM, pair kernel (path 9)
cat > /tmp/one_linear.py <<'PY'
import sys
sys.path.insert(0, ".")
import pipo_synth as synth
from paper_2504_03664_b200 import pipo
shape = synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64)
pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
print(pipo.pipo_bench_linear(pl.ctx, 1, int(sys.argv[1]), 64, int(sys.argv[2]) if len(sys.argv) > 2 else 21504, int(sys.argv[3]) if len(sys.argv) > 3 else 7168, 3))
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_pair_kernel -s 6 -c 1 -o gpurun_out/ncu_pair_qkv python /tmp/one_linear.py 9 28672 7168 > gpurun_out/ncu_pair.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu_pair.log
