import os, sys
sys.path.insert(0, ".")
import pipo_synth as synth
from paper_2504_03664_b200 import pipo
shape = synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64)
pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
for fix in ("0", "1"):
    os.environ["PIPO_TM_FIXUP"] = fix
    for name, M, N, K in [("c5_qkv", 64, 21504, 7168), ("c5_out", 64, 7168, 7168)]:
        print(f"== fix {fix} {name}", file=sys.stderr, flush=True)
        us = pipo.pipo_bench_linear(pl.ctx, 1, pipo.PATH_TM, M, N, K, 10)
        print(f"{name} fix {fix}: {us:.2f} us", file=sys.stderr, flush=True)
