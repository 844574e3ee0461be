"""Causal prefill attention timing at the configs' prompt shapes: tcgen05 (variant 0),
mma.sync (2) and CUDA cores (1); TFLOP/s count 4 * b * H * (n^2 / 2) * hd (QK^T and PV,
causal half)."""
import sys
sys.path.insert(0, ".")
import pipo_synth as synth
from paper_2504_03664_b200 import pipo
pl = pipo.Pipeline(pipo.make_config(synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64), max_batch=4, max_seq=16,
                                    weight_tier=pipo.PIPO_TIER_DEVICE))
cases = [("c5", 64, 512, 7168, 56, 0), ("c3", 32, 512, 4096, 32, 0), ("c2", 16, 256, 2048, 32, 0),
         ("c6", 64, 512, 4096, 32, 8), ("c4", 64, 512, 5120, 40, 0)]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0] in sys.argv[1:]]
for name, b, n, d, H, Hkv in cases:
    hd = d // H
    fl = 4 * b * H * (n * n / 2) * hd
    row = {}
    for v, nm in ((0, "tcgen05"), (2, "mma_sync")):
        us = pipo.pipo_bench_attention_prefill(pl.ctx, b, n, d, H, v, 5, Hkv)
        row[nm] = (round(us, 1), round(fl / us / 1e6, 1))
    print(name, "us, TFLOP/s:", row, flush=True)
