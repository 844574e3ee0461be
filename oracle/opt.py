"""OPT decoder forward in float64 — oracle (TEST INFRASTRUCTURE ONLY).

The computation the offloading pipeline must reproduce (SURVEY.md §8(c) steps
2-5).  The paper names the model (OPT, §4.1) and the task split
("Computation encompasses MHA and MLP layers, as well as the input and output
embedding layers", §3.1.2) but not the block itself; the OPT
block below is [ext] transformers' `modeling_opt.py` (pre-LN for 125M..30B):

  embed     h[t] = E_tok[id_t] + E_pos[past + t + 2]
  per layer x = LN(h; g1, b1)                    (biased variance, eps 1e-5)
            [q|k|v] = x W_qkv^T + b_qkv;  q *= hd^-0.5   (after the bias)
            append k, v at positions past .. past+n-1      (the KV cache)
            o_head = softmax(q K^T) V   over positions <= own (causal)
            h += o W_out^T + b_out
            x = LN(h; g2, b2);  h += relu(x W_fc1^T + b_fc1) W_fc2^T + b_fc2
  head      logits = LN(h; gf, bf) E_tok^T     (tied, no bias)
  greedy    next = argmax(logits), lowest index on ties (np.argmax)

Weights are the int4 path's dequantized weights (oracle/quant.py) or the fp16
masters, held in float64; all arithmetic is float64, one library matmul per
product, no blocking or reordering beyond the definitions above.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import quant

LN_EPS = 1e-5
POS_OFFSET = 2          # [ext] OPTLearnedPositionalEmbedding offset


def layer_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray) -> np.ndarray:
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + LN_EPS) * g + b


def softmax(s: np.ndarray) -> np.ndarray:
    m = s.max(axis=-1, keepdims=True)
    e = np.exp(s - m)
    return e / e.sum(axis=-1, keepdims=True)


def attention(q, k_all, v_all, past: int, n_heads: int) -> np.ndarray:
    """q [b, n, d] (already scaled); k_all, v_all [b, past+n, d].
    Query t (absolute position past+t) attends to positions 0..past+t."""
    b, n, d = q.shape
    hd = d // n_heads
    L = past + n
    qh = q.reshape(b, n, n_heads, hd).transpose(0, 2, 1, 3)          # [b,H,n,hd]
    kh = k_all[:, :L].reshape(b, L, n_heads, hd).transpose(0, 2, 1, 3)
    vh = v_all[:, :L].reshape(b, L, n_heads, hd).transpose(0, 2, 1, 3)
    s = qh @ kh.transpose(0, 1, 3, 2)                                  # [b,H,n,L]
    allowed = np.arange(L)[None, :] <= (past + np.arange(n))[:, None]  # [n, L]
    s = np.where(allowed[None, None], s, -np.inf)
    p = softmax(s)
    o = p @ vh                                                         # [b,H,n,hd]
    return o.transpose(0, 2, 1, 3).reshape(b, n, d)


@dataclass
class LayerW:
    ln1_g: np.ndarray
    ln1_b: np.ndarray
    w_qkv: np.ndarray      # [3d, d] rows q | k | v
    b_qkv: np.ndarray
    w_out: np.ndarray      # [d, d]
    b_out: np.ndarray
    ln2_g: np.ndarray
    ln2_b: np.ndarray
    w_fc1: np.ndarray      # [F, d]
    b_fc1: np.ndarray
    w_fc2: np.ndarray      # [d, F]
    b_fc2: np.ndarray


MATRICES = ("w_qkv", "w_out", "w_fc1", "w_fc2")


def layer_from_masters(m: dict, wfmt: str) -> LayerW:
    """wfmt 'int4': the four linear weights are quantize->dequantize'd; everything
    else (biases, LN) stays at its fp16-exact master value.  'fp16': masters."""
    kw = {}
    for k, v in m.items():
        v = np.asarray(v, dtype=np.float32)
        if k in MATRICES and wfmt == "int4":
            v = quant.quant_dequant(v)
        elif wfmt not in ("int4", "fp16"):
            raise ValueError(wfmt)
        kw[k] = v.astype(np.float64)
    return LayerW(**kw)


def kv_quant_dequant(x: np.ndarray) -> np.ndarray:
    """INT4 KV cache ("quantizing both weights and KV-cache to INT4";
    reading Q17/NEXT-2): every cached row is stored with the weights' encoding —
    groups of 64 consecutive features (inside one head for hd in {64, 128}), fp16
    scale = absmax/7 — and read back as q * s."""
    shp = x.shape
    flat = np.asarray(x, dtype=np.float32).reshape(-1, shp[-1])
    return quant.quant_dequant(flat).reshape(shp).astype(np.float64)


def decoder_layer(h: np.ndarray, w: LayerW, kc: np.ndarray, vc: np.ndarray,
                  past: int, n_heads: int, kv_int4: bool = False) -> np.ndarray:
    """h [b, n, d] float64; kc/vc [b, s_max, d] float64 caches (written at past..).
    kv_int4: the cache holds int4-g64 quantize->dequantize'd rows; a multi-token
    pass (prefill) attends over its freshly computed K/V, a decode step reads the
    cache (its own new row included) — reading Q17b in DESIGN.md."""
    b, n, d = h.shape
    hd = d // n_heads
    x = layer_norm(h, w.ln1_g, w.ln1_b)
    qkv = x @ w.w_qkv.T + w.b_qkv
    q = qkv[..., :d] * (hd ** -0.5)
    k_new, v_new = qkv[..., d:2 * d], qkv[..., 2 * d:]
    if kv_int4:
        kc[:, past:past + n] = kv_quant_dequant(k_new)
        vc[:, past:past + n] = kv_quant_dequant(v_new)
    else:
        kc[:, past:past + n] = k_new
        vc[:, past:past + n] = v_new
    if kv_int4 and n > 1:
        if past != 0:
            raise ValueError("int4-KV multi-token pass only at past = 0 (prefill)")
        o = attention(q, k_new, v_new, 0, n_heads)
    else:
        o = attention(q, kc, vc, past, n_heads)
    h = h + o @ w.w_out.T + w.b_out
    x = layer_norm(h, w.ln2_g, w.ln2_b)
    u = np.maximum(x @ w.w_fc1.T + w.b_fc1, 0.0)
    return h + u @ w.w_fc2.T + w.b_fc2


@dataclass
class OracleOPT:
    """Whole-model oracle with its own KV cache (b sequences, equal length)."""
    n_heads: int
    tok: np.ndarray
    pos: np.ndarray
    lnf_g: np.ndarray
    lnf_b: np.ndarray
    layers: list
    s_max: int
    past: int = 0
    kv_int4: bool = False
    kc: list = field(default_factory=list)
    vc: list = field(default_factory=list)
    capture: list = field(default_factory=list)   # per-layer outputs of the last call

    @classmethod
    def from_masters(cls, n_heads, embed: dict, layer_masters: list, wfmt: str, s_max: int, kv_int4: bool = False):
        return cls(n_heads=n_heads, kv_int4=kv_int4,
                   tok=embed["tok"].astype(np.float64), pos=embed["pos"].astype(np.float64),
                   lnf_g=embed["lnf_g"].astype(np.float64), lnf_b=embed["lnf_b"].astype(np.float64),
                   layers=[layer_from_masters(m, wfmt) for m in layer_masters], s_max=s_max)

    def embed(self, ids: np.ndarray) -> np.ndarray:
        b, n = ids.shape
        positions = self.past + np.arange(n) + POS_OFFSET
        return self.tok[ids] + self.pos[positions][None]

    def head(self, h_last: np.ndarray) -> np.ndarray:
        return layer_norm(h_last, self.lnf_g, self.lnf_b) @ self.tok.T

    def forward(self, ids: np.ndarray, all_logits: bool = False) -> np.ndarray:
        ids = np.asarray(ids)
        b, n = ids.shape
        if self.past == 0:
            d = self.tok.shape[1]
            self.kc = [np.zeros((b, self.s_max, d)) for _ in self.layers]
            self.vc = [np.zeros((b, self.s_max, d)) for _ in self.layers]
        if self.past + n > self.s_max:
            raise ValueError("sequence exceeds s_max")
        h = self.embed(ids)
        self.capture = []
        for j, w in enumerate(self.layers):
            h = decoder_layer(h, w, self.kc[j], self.vc[j], self.past, self.n_heads, self.kv_int4)
            self.capture.append(h.copy())
        self.past += n
        return self.head(h) if all_logits else self.head(h[:, -1])

    def prefill(self, ids: np.ndarray) -> np.ndarray:
        self.past = 0
        return self.forward(ids)

    def decode(self, ids: np.ndarray) -> np.ndarray:
        return self.forward(np.asarray(ids).reshape(-1, 1))


def greedy(logits: np.ndarray) -> np.ndarray:
    """argmax per row, lowest index on exact ties."""
    return np.argmax(logits, axis=-1).astype(np.int32)


def generate(model: OracleOPT, prompt: np.ndarray, gen: int):
    """Greedy generation: prefill emits token 1, then gen-1 decode steps
    (reading Q21).  Returns (ids [b, gen], per-step logits list)."""
    logits = [model.prefill(prompt)]
    ids = [greedy(logits[-1])]
    for _ in range(gen - 1):
        logits.append(model.decode(ids[-1]))
        ids.append(greedy(logits[-1]))
    return np.stack(ids, axis=1), logits
