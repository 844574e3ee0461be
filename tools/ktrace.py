"""CUPTI (torch.profiler) trace of isolated linear launches: per-kernel durations and the
gaps between consecutive kernels (main GEMM -> stream-K reduce -> next GEMM).

    python tools/ktrace.py c5_qkv c5_out
"""
import collections
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import pipo_synth as synth  # noqa: E402
from paper_2504_03664_b200 import pipo  # noqa: E402

CASES = {"c5_qkv": (64, 21504, 7168), "c5_out": (64, 7168, 7168), "c5_fc1": (64, 28672, 7168),
         "c5_fc2": (64, 7168, 28672), "c6_fc2": (64, 4096, 14336)}
shape = synth.OPTShape(256, 1, 4, 512, vocab=512, max_pos=64)
pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
out = {}
for name in sys.argv[1:] or list(CASES):
    M, N, K = CASES[name]
    pipo.pipo_bench_linear(pl.ctx, 1, pipo.PATH_TM, M, N, K, 3)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        pipo.pipo_bench_linear(pl.ctx, 1, pipo.PATH_TM, M, N, K, 10)
        torch.cuda.synchronize()
    ev = sorted((e.time_range.start, e.time_range.end, e.name.split("(")[0].replace("void pipo::", "")[:40])
                for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA)
    dur = collections.defaultdict(list)
    gaps = collections.defaultdict(list)
    for s, e, n in ev:
        dur[n].append(e - s)
    for (s0, e0, n0), (s1, e1, n1) in zip(ev, ev[1:]):
        gaps[f"{n0[:18]} -> {n1[:18]}"].append(s1 - e0)
    out[name] = {"dur_us": {k: round(float(np.median(v)), 2) for k, v in dur.items()},
                 "gap_us": {k: round(float(np.median(v)), 2) for k, v in gaps.items()}}
    print(name, json.dumps(out[name]), flush=True)
json.dump(out, open("gpurun_out/ktrace.json", "w"), indent=1)
