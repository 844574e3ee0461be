"""Decode-attention kernel timing at the configs' shapes (cold HBM: KV copies rotate).
MHA (OPT c1-c5) and GQA (LLaMA c6-c8) with the production kernel choice, plus the
CUDA-core variants for reference."""
import sys
sys.path.insert(0, ".")
import pipo_synth as synth
from paper_2504_03664_b200 import pipo
pl = pipo.Pipeline(pipo.make_config(synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64), max_batch=4, max_seq=16,
                                    weight_tier=pipo.PIPO_TIER_DEVICE))
cases = [("c5", 64, 528, 7168, 56, 0), ("c3", 32, 528, 4096, 32, 0), ("c2", 16, 272, 2048, 32, 0),
         ("c6", 64, 528, 4096, 32, 8), ("c6_L1040", 64, 1040, 4096, 32, 8), ("c7", 1, 528, 4096, 32, 8),
         ("c8", 64, 528, 2048, 32, 8)]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0] in sys.argv[1:]]
for name, b, L, d, H, Hkv in cases:
    row = {}
    dkv = d // H * (Hkv or H)
    for v in ([0, 1] if not Hkv else [0, 5, 6, 3]):
        us = pipo.pipo_bench_attention(pl.ctx, b, L, d, H, v, 20, Hkv)
        row[f"var{v}"] = (round(us, 2), round(2 * L * b * dkv * 2 / us / 1e3, 1))
    print(name, "us, GB/s:", row, flush=True)
