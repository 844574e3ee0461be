"""Prefill GEMM timing: tcgen05 tile kernel v1 vs the TMEM-A prefill kernel's tile
configurations (PIPO_TP_CFG) at the OPT prefill shapes (M = b * P)."""
import json
import os
import sys

sys.path.insert(0, ".")
import pipo_synth as synth  # noqa: E402
from paper_2504_03664_b200 import pipo  # noqa: E402

shape = synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64)
pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
cases = [("pre_c5_qkv", 32768, 21504, 7168), ("pre_c5_out", 32768, 7168, 7168), ("pre_c5_fc1", 32768, 28672, 7168),
         ("pre_c5_fc2", 32768, 7168, 28672), ("pre_c2_qkv", 4096, 6144, 2048), ("pre_c3_fc1", 16384, 16384, 4096)]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0] in sys.argv[1:]]
cfgs = os.environ.get("TP_CFGS", "0,1,2,3,4").split(",")
for name, M, N, K in cases:
    res = {}
    runs = [("tc_v1", pipo.PATH_TC, None)] + [(f"tp{c}", pipo.PATH_TP, c) for c in cfgs]
    for label, p, c in runs:
        if c is not None:
            os.environ["PIPO_TP_CFG"] = c
        try:
            us = pipo.pipo_bench_linear(pl.ctx, 1, p, M, N, K, 5)
            res[label] = {"us": round(us, 1), "TFLOPs": round(2 * M * N * K / us / 1e6, 1)}
        except pipo.PipoError as e:
            res[label] = str(e)
    print(name, json.dumps(res), flush=True)
