"""Decode-GEMM variants at the c5 shapes: time (events, 10 cold launches) per
(PIPO_TM_CFG, PIPO_TM_FIXUP) and check each variant is bit-identical to the default."""
import json
import os
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import pipo_synth as synth  # noqa: E402
from paper_2504_03664_b200 import pipo  # noqa: E402

shape = synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64)
pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
cases = [("c5_qkv", 64, 21504, 7168), ("c5_out", 64, 7168, 7168), ("c5_fc1", 64, 28672, 7168),
         ("c5_fc2", 64, 7168, 28672), ("c6_qkv", 64, 6144, 4096), ("c2_fc1", 16, 8192, 2048)]
variants = [v.split(":") for v in (sys.argv[1:] or ["6:0", "6:2", "7:0", "8:0", "9:0", "7:2", "8:2"])]
rng = np.random.default_rng(0)
res = {}
for name, M, N, K in cases:
    x = rng.standard_normal((M, K), dtype=np.float32).astype(np.float16)
    w = (rng.standard_normal((N, K), dtype=np.float32) * 0.02).astype(np.float32)
    ref = None
    row = {}
    for cfg, fix in variants:
        os.environ["PIPO_TM_CFG"], os.environ["PIPO_TM_FIXUP"] = cfg, fix
        y = pipo.pipo_linear(pl.ctx, 1, pipo.PATH_TM, x, w)
        if ref is None:
            ref = y
        same = bool(np.array_equal(y, ref))
        us = pipo.pipo_bench_linear(pl.ctx, 1, pipo.PATH_TM, M, N, K, 20)
        row[f"{cfg}:{fix}"] = {"us": round(us, 2), "bit_identical": same}
    res[name] = row
    print(name, json.dumps(row), flush=True)
json.dump(res, open("gpurun_out/tm_variants.json", "w"), indent=1)
