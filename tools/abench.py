"""Decode-attention kernel timing at the configs' shapes (v2 production vs v1)."""
import sys
sys.path.insert(0, ".")
import pipo_synth as synth
from paper_2504_03664_b200 import pipo
pl = pipo.Pipeline(pipo.make_config(synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64), max_batch=4, max_seq=16,
                                    weight_tier=pipo.PIPO_TIER_DEVICE))
for name, b, L, d, H in [("c5", 64, 528, 7168, 56), ("c4", 64, 528, 5120, 40), ("c3", 32, 528, 4096, 32),
                         ("c2", 16, 272, 2048, 32), ("c1", 4, 36, 768, 12)]:
    row = {}
    for v in (0, 1):
        us = pipo.pipo_bench_attention(pl.ctx, b, L, d, H, v, 10)
        row[f"v{v + 1}"] = (round(us, 2), round(2 * L * b * d * 2 / us / 1e3, 1))
    print(name, "us, GB/s:", row, flush=True)
