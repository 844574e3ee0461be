"""Isolated kernel timing of the linear-layer paths at the OPT decode/prefill shapes."""
import json
import sys

sys.path.insert(0, ".")
import pipo_synth as synth  # noqa: E402
from paper_2504_03664_b200 import pipo  # noqa: E402

shape = synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64)
pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
paths = {"gemm_mma": pipo.PATH_GEMM, "tc_v1": pipo.PATH_TC, "ws": pipo.PATH_WS, "tm": pipo.PATH_TM,
         "gemv": pipo.PATH_GEMV, "head": pipo.PATH_HEAD, "pair": pipo.PATH_PAIR}
import os
if os.environ.get("KBENCH_PATHS"):
    paths = {k: v for k, v in paths.items() if k in os.environ["KBENCH_PATHS"].split(",")}
cases = [("c5_qkv", 64, 21504, 7168), ("c5_out", 64, 7168, 7168), ("c5_fc1", 64, 28672, 7168),
         ("c5_fc2", 64, 7168, 28672), ("c2_qkv", 16, 6144, 2048), ("c2_fc2", 16, 2048, 8192),
         ("c3_qkv", 32, 12288, 4096), ("pre_c2_qkv", 4096, 6144, 2048), ("c5_head", 64, 50272, 7168),
         ("c6_head", 64, 128256, 4096), ("c6_qkv", 64, 6144, 4096), ("c6_fc1", 64, 28672, 4096), ("c6_fc2", 64, 4096, 14336),
         ("c7_qkv", 1, 6144, 4096), ("c7_fc1", 1, 28672, 4096),
         ("c7_fc2", 1, 4096, 14336), ("c1_fc1", 4, 3072, 768)]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0] in sys.argv[1:]]
out = {}
for name, M, N, K in cases:
    wbytes = N * K / 2 + N * K / 32
    res = {}
    for pn, p in paths.items():
        try:
            wf = int(os.environ.get("KBENCH_WFMT", "1"))
            wb = wbytes if wf == 1 else N * K * 2
            us = pipo.pipo_bench_linear(pl.ctx, wf, p, M, N, K, 10)
            res[pn] = {"us": round(us, 2), "GBs": round(wb / us / 1e3, 1),
                       "TFLOPs": round(2 * M * N * K / us / 1e6, 1)}
        except pipo.PipoError as e:
            res[pn] = str(e)
    out[name] = res
    print(name, json.dumps(res), flush=True)
json.dump(out, open("gpurun_out/kbench.json", "w"), indent=1)
