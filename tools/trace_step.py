"""CUPTI (torch.profiler) trace of live decode steps: true per-kernel GPU start/end
timestamps with the copy stream running concurrently (ncu serialises everything).
Reports per-kernel average duration, and for the linear-layer launches the gap from the
previous kernel on the compute stream.

    python tools/trace_step.py --config c5 --tier host --steps 2
"""
import argparse
import collections
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import pipo_synth as synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2504_03664_b200 import pipo  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--tier", default="host", choices=["host", "device"])
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--kprof", type=int, default=1)
args = ap.parse_args()
c = CONFIGS[args.config]
s, b, P = c["shape"], c["b"], c["P"]
flags = pipo.PIPO_F_TIMELINE | (pipo.PIPO_F_KPROF if args.kprof else 0)
cfg = pipo.make_config(s, max_batch=b, max_seq=P + 8, weight_tier=1 if args.tier == "host" else 0,
                       kv_tier=0, flags=flags)
pl = pipo.Pipeline(cfg)
pl.load_synthetic(pipo.PIPO_LAYER_EMBED, synth.WEIGHT_SEED)
for j in range(s.n_layers):
    pl.load_synthetic(j, synth.WEIGHT_SEED)
nxt, _ = pl.prefill(synth.prompts(b, P, s.vocab))
for _ in range(2):
    nxt, _ = pl.decode_step(nxt)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(args.steps):
        nxt, _ = pl.decode_step(nxt)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = [(e.time_range.start, e.time_range.end, e.name) for e in ev]
kern.sort()
dur = collections.defaultdict(list)
for st, en, nm in kern:
    dur[nm.split("(")[0][:50]].append(en - st)
out = {k: {"n": len(v), "avg_us": float(np.mean(v)), "total_ms": float(np.sum(v)) / 1e3} for k, v in dur.items()}
# gaps before gemm_tm launches (previous compute-stream kernel end -> this start)
comp = [k for k in kern if "Memcpy" not in k[2] and "memcpy" not in k[2]]
gaps = []
for (s0, e0, n0), (s1, e1, n1) in zip(comp, comp[1:]):
    if "gemm_tm" in n1:
        gaps.append(s1 - e0)
out["_gap_before_gemm_tm_us"] = {"avg": float(np.mean(gaps)) if gaps else None,
                                "p50": float(np.median(gaps)) if gaps else None, "n": len(gaps)}
# gap statistics by (previous kernel -> next kernel) pair on the compute stream
pairs = collections.defaultdict(list)
short = lambda n: n.split("(")[0].replace("void pipo::", "").replace("pipo::", "")[:28]
for (s0, e0, n0), (s1, e1, n1) in zip(comp, comp[1:]):
    pairs[f"{short(n0)} -> {short(n1)}"].append(s1 - e0)
out["_gaps_by_pair_us"] = {k: {"n": len(v), "avg": float(np.mean(v)), "p50": float(np.median(v))}
                          for k, v in sorted(pairs.items(), key=lambda kv: -np.sum(kv[1]))[:12]}
span = (kern[-1][1] - kern[0][0]) / 1e3 if kern else 0
out["_span_ms"] = span
print(json.dumps({"config": args.config, "tier": args.tier, "kernels": out}, indent=1))
