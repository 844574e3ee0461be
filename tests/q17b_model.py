"""Hand-built one-layer OPT model that separates the two readings of an INT4 KV
cache at a decode step (reading Q17b; the paper only says "quantizing both
weights and KV-cache to INT4"):

  A (taken): the decode step appends its new K/V row quantized and attends over the
             int4 cache, its OWN row included (dequantized);
  B:         the decode step attends over the quantized old rows plus its own row
             in full precision.

Construction (d = 64, one head, F = 64, no position table, zero biases):
  * q and k projections are zero -> every score is 0 -> softmax is exactly uniform;
  * the v projection and the out-projection are the identity (int4: 0.99976 I);
  * FC1 / FC2 are zero, LayerNorms are plain (g = 1, b = 0);
  * the decode token's embedding is a spike 3 e_0: LN turns it into one element
    ~7.94 and 63 elements ~-0.126, and the int4 encoding (scale = absmax / 7) rounds
    those 63 to 0.  Under A the decode output moves by v/2 with those 63 entries 0,
    under B by -0.063 each: a 0.063 absolute difference against fp16 errors ~1e-3;
  * the prompt token is the spike 3 e_1, so every cached code is far from a rounding
    boundary (the spike codes are exactly +-7, the rest |x / s| ~ 0.11 -> 0): fp16 vs
    fp64 K/V values cannot flip a code, which they would for a generic row (one flip
    moves an output element by s / 2).
Only weights live here (no method arithmetic)."""
from __future__ import annotations

import numpy as np

import pipo_synth as synth

SHAPE = synth.OPTShape(d_model=64, n_layers=1, n_heads=1, ffn_dim=64, vocab=64, max_pos=16)
PROMPT_TOKEN, SPIKE_TOKEN = 5, 9


def masters():
    d, F, V = SHAPE.d_model, SHAPE.ffn_dim, SHAPE.vocab
    rng = np.random.default_rng(17)
    tok = rng.standard_normal((V, d)).astype(np.float16).astype(np.float32)
    tok[SPIKE_TOKEN] = 0.0
    tok[SPIKE_TOKEN, 0] = 3.0
    tok[PROMPT_TOKEN] = 0.0
    tok[PROMPT_TOKEN, 1] = 3.0
    emb = {"tok": tok, "pos": np.zeros((SHAPE.max_pos + 2, d), np.float32),
           "lnf_g": np.ones(d, np.float32), "lnf_b": np.zeros(d, np.float32)}
    w_qkv = np.zeros((3 * d, d), np.float32)
    w_qkv[2 * d:] = np.eye(d, dtype=np.float32)
    layer = {"ln1_g": np.ones(d, np.float32), "ln1_b": np.zeros(d, np.float32),
             "w_qkv": w_qkv, "b_qkv": np.zeros(3 * d, np.float32),
             "w_out": np.eye(d, dtype=np.float32), "b_out": np.zeros(d, np.float32),
             "ln2_g": np.ones(d, np.float32), "ln2_b": np.zeros(d, np.float32),
             "w_fc1": np.zeros((F, d), np.float32), "b_fc1": np.zeros(F, np.float32),
             "w_fc2": np.zeros((d, F), np.float32), "b_fc2": np.zeros(d, np.float32)}
    return emb, [layer]


def prompt(b: int = 2) -> np.ndarray:
    return np.full((b, 1), PROMPT_TOKEN, np.int32)


def decode_tokens(b: int = 2) -> np.ndarray:
    return np.full(b, SPIKE_TOKEN, np.int32)
