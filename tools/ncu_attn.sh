# ncu --set full of the decode attention kernels at c5 (MHA) and c6 (GQA, tensor cores), cold HBM
cat > /tmp/one_attn.py <<'PY'
import sys
sys.path.insert(0, ".")
import pipo_synth as synth
from paper_2504_03664_b200 import pipo
pl = pipo.Pipeline(pipo.make_config(synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64), max_batch=4, max_seq=16,
                                    weight_tier=pipo.PIPO_TIER_DEVICE))
b, L, d, H, Hkv = [int(x) for x in sys.argv[1:6]]
print(pipo.pipo_bench_attention(pl.ctx, b, L, d, H, 0, 4, Hkv))
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 6 -c 1 -o gpurun_out/ncu_attn_c6 python /tmp/one_attn.py 64 528 4096 32 8 > gpurun_out/ncu_attn_c6.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 6 -c 1 -o gpurun_out/ncu_attn_c5 python /tmp/one_attn.py 64 528 7168 56 0 > gpurun_out/ncu_attn_c5.log 2>&1
timeout 300 python tools/abench.py > gpurun_out/abench.log 2>&1
echo done
