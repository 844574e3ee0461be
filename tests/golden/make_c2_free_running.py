"""Write tests/golden/c2_free_running.json from the ORACLE only (oracle/opt.py).

configs[1] (OPT-1.3B, 24 layers, b = 16, P = 256, gen 32; BASELINE.json) generated
free-running and greedily by the fp64 oracle on the seeded synthetic weights and
prompts (pipo_synth, seeds 2504 / 3664).  Stored per sequence: the 32 greedy ids
and, per step, the oracle's top-1 minus top-2 logit margin.  The GPU test
(`tests/test_gpu_fullsize.py::test_c2_free_running_greedy_ids`) uses the margins to
pick the sequences whose every step is decided by a wide margin (reading Q11: "the
committed fixture ... chosen so that free-running greedy ids match exactly"), re-runs
the oracle live for those sequences and asserts exact id equality.

    python tests/golden/make_c2_free_running.py      # ~5 min on 8 cores, ~12 GB RAM
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import pipo_synth as synth  # noqa: E402
from oracle import opt  # noqa: E402

B, P, G = 16, 256, 32


def main():
    s = synth.OPT_1_3B
    t0 = time.time()
    emb = synth.embed_masters(s)
    layers = [opt.layer_from_masters(synth.layer_masters(s, j), "int4") for j in range(s.n_layers)]
    model = opt.OracleOPT(n_heads=s.n_heads, tok=emb["tok"].astype(np.float64), pos=emb["pos"].astype(np.float64),
                          lnf_g=emb["lnf_g"].astype(np.float64), lnf_b=emb["lnf_b"].astype(np.float64),
                          layers=layers, s_max=P + G)
    prompt = synth.prompts(B, P, s.vocab)
    ids, logits = opt.generate(model, prompt, G)
    margins = []
    for lg in logits:
        srt = np.sort(lg, axis=-1)
        margins.append(srt[:, -1] - srt[:, -2])
    margins = np.stack(margins, 1)                       # [B, G]
    out = {
        "source": "tests/golden/make_c2_free_running.py (oracle/opt.py fp64, int4-g64 weights; pipo_synth seeds "
                  f"{synth.WEIGHT_SEED}/{synth.PROMPT_SEED})",
        "config": {"model": "OPT-1.3B", "b": B, "P": P, "G": G},
        "ids": ids.tolist(),
        "margins": margins.tolist(),
        "logit_absmax": float(max(np.abs(lg).max() for lg in logits)),
        "seconds": time.time() - t0,
    }
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c2_free_running.json")
    json.dump(out, open(path, "w"))
    print(path, "min margin per sequence:", np.round(margins.min(1), 4).tolist(), f"{time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
