"""LLaMA3.1 decoder forward in float64 — oracle (TEST INFRASTRUCTURE ONLY).

NEXT-4 of SURVEY.md §8(f): the paper's second model family.  The paper evaluates
LLaMA3.1-8B/70B (§4.1, Figs. 9/10, the latency table)
and writes its memory model for it (§3.5): grouped-query attention
with h heads and h_kv KV heads, an MLP of hidden width d_h with three
d x d_h matrices (W_mlp = p d (3 d_h + 1)), K and V each d h_kv/h wide
(C = 2 p b s l d h_kv/h).  The block itself is [ext] transformers'
`modeling_llama.py` (Llama-3.1 configs):

  embed     h[t] = E_tok[id_t]                               (no position table)
  per layer x = RMS(h; g1) = h / sqrt(mean(h^2) + eps) * g1   (eps 1e-5)
            q = x Wq^T, k = x Wk^T, v = x Wv^T                (no biases; W_qkv rows q|k|v)
            q, k rotated by RoPE at their absolute position p (rotate-half pairs
              (i, i + hd/2), angle p * inv_freq[i], llama3 frequency rule below)
            q *= hd^-0.5
            append k, v at positions past .. past+n-1
            query head j attends with KV head j // (h / h_kv)   (GQA), causal softmax
            h += o Wo^T
            x = RMS(h; g2);  h += (silu(x Wg^T) * (x Wu^T)) Wd^T   (SwiGLU; W_fc1 rows gate|up)
  head      logits = RMS(h; gf) W_lm^T                          (untied LM head)
  greedy    next = argmax(logits), lowest index on ties

llama3 inverse frequencies ([ext] transformers `_compute_llama3_parameters`):
  inv_i = theta^(-2i/hd);  wavelen_i = 2 pi / inv_i
  wavelen > orig/low_f  -> inv_i / factor
  wavelen < orig/high_f -> inv_i
  otherwise             -> (1 - sm) inv_i / factor + sm inv_i,  sm = (orig/wavelen - low_f) / (high_f - low_f)

Weights are the int4 path's dequantized weights (oracle/quant.py) or the fp16 masters
in float64; all arithmetic is float64, one library matmul per product.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import quant

RMS_EPS = 1e-5


def rms_norm(x: np.ndarray, g: np.ndarray, eps: float = RMS_EPS) -> np.ndarray:
    return x / np.sqrt((x * x).mean(axis=-1, keepdims=True) + eps) * g


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def rope_inv_freq(hd: int, theta: float, factor: float = 0.0, low_freq: float = 1.0, high_freq: float = 4.0,
                  orig_max_pos: int = 8192) -> np.ndarray:
    """[hd/2] float64 inverse frequencies; factor == 0 -> plain RoPE (no llama3 rule)."""
    inv = 1.0 / theta ** (np.arange(0, hd, 2, dtype=np.float64) / hd)
    if not factor:
        return inv
    low_wl, high_wl = orig_max_pos / low_freq, orig_max_pos / high_freq
    wl = 2.0 * math.pi / inv
    out = np.where(wl > low_wl, inv / factor, inv)
    sm = (orig_max_pos / wl - low_freq) / (high_freq - low_freq)
    smoothed = (1.0 - sm) * out / factor + sm * out
    medium = ~(wl < high_wl) & ~(wl > low_wl)
    return np.where(medium, smoothed, out)


def rope(x: np.ndarray, positions: np.ndarray, inv_freq: np.ndarray) -> np.ndarray:
    """x [b, n, heads, hd]; positions [n] absolute.  Rotate-half convention:
    out[:half] = x1 cos - x2 sin, out[half:] = x2 cos + x1 sin, angle = p * inv_freq."""
    half = x.shape[-1] // 2
    ang = positions.astype(np.float64)[:, None] * inv_freq[None, :]      # [n, half]
    c, s = np.cos(ang)[None, :, None, :], np.sin(ang)[None, :, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def attention_gqa(q, k_all, v_all, past: int, n_heads: int, n_kv_heads: int) -> np.ndarray:
    """q [b, n, h*hd] (scaled, rotated); k_all, v_all [b, past+n, h_kv*hd].
    Query head j uses KV head j // (h / h_kv); query t (position past+t) sees 0..past+t."""
    b, n, dq = q.shape
    hd = dq // n_heads
    group = n_heads // n_kv_heads
    L = past + n
    qh = q.reshape(b, n, n_heads, hd).transpose(0, 2, 1, 3)                    # [b,h,n,hd]
    kh = k_all[:, :L].reshape(b, L, n_kv_heads, hd).transpose(0, 2, 1, 3)      # [b,hkv,L,hd]
    vh = v_all[:, :L].reshape(b, L, n_kv_heads, hd).transpose(0, 2, 1, 3)
    kh = np.repeat(kh, group, axis=1)                                          # head j -> kv j//group
    vh = np.repeat(vh, group, axis=1)
    s = qh @ kh.transpose(0, 1, 3, 2)
    allowed = np.arange(L)[None, :] <= (past + np.arange(n))[:, None]
    s = np.where(allowed[None, None], s, -np.inf)
    m = s.max(axis=-1, keepdims=True)
    e = np.exp(s - m)
    p = e / e.sum(axis=-1, keepdims=True)
    return (p @ vh).transpose(0, 2, 1, 3).reshape(b, n, dq)


@dataclass
class LlamaLayerW:
    ln1_g: np.ndarray
    w_qkv: np.ndarray      # [d + 2 d_kv, d] rows q | k | v
    w_out: np.ndarray      # [d, d]
    ln2_g: np.ndarray
    w_fc1: np.ndarray      # [2F, d] rows gate | up
    w_fc2: np.ndarray      # [d, F]


MATRICES = ("w_qkv", "w_out", "w_fc1", "w_fc2")


def layer_from_masters(m: dict, wfmt: str) -> LlamaLayerW:
    kw = {}
    for k, v in m.items():
        v = np.asarray(v, dtype=np.float32)
        if k in MATRICES and wfmt == "int4":
            v = quant.quant_dequant(v)
        elif wfmt not in ("int4", "fp16"):
            raise ValueError(wfmt)
        kw[k] = v.astype(np.float64)
    return LlamaLayerW(**kw)


def decoder_layer(h, w: LlamaLayerW, kc, vc, past: int, n_heads: int, n_kv_heads: int, inv_freq) -> np.ndarray:
    """h [b, n, d] float64; kc/vc [b, s_max, d_kv] float64 caches (written at past..)."""
    b, n, d = h.shape
    hd = d // n_heads
    dkv = n_kv_heads * hd
    x = rms_norm(h, w.ln1_g)
    qkv = x @ w.w_qkv.T
    pos = past + np.arange(n)
    q = rope(qkv[..., :d].reshape(b, n, n_heads, hd), pos, inv_freq).reshape(b, n, d) * (hd ** -0.5)
    k_new = rope(qkv[..., d:d + dkv].reshape(b, n, n_kv_heads, hd), pos, inv_freq).reshape(b, n, dkv)
    v_new = qkv[..., d + dkv:]
    kc[:, past:past + n] = k_new
    vc[:, past:past + n] = v_new
    o = attention_gqa(q, kc, vc, past, n_heads, n_kv_heads)
    h = h + o @ w.w_out.T
    x = rms_norm(h, w.ln2_g)
    F = w.w_fc2.shape[1]
    gu = x @ w.w_fc1.T
    return h + (silu(gu[..., :F]) * gu[..., F:]) @ w.w_fc2.T


@dataclass
class OracleLlama:
    """Whole-model oracle with its own KV cache (b sequences, equal length)."""
    n_heads: int
    n_kv_heads: int
    inv_freq: np.ndarray
    tok: np.ndarray
    lnf_g: np.ndarray
    lm_head: np.ndarray
    layers: list
    s_max: int
    past: int = 0
    kc: list = field(default_factory=list)
    vc: list = field(default_factory=list)
    capture: list = field(default_factory=list)

    @classmethod
    def from_masters(cls, shape, embed: dict, layer_masters: list, wfmt: str, s_max: int):
        inv = rope_inv_freq(shape.head_dim, shape.rope_theta, shape.rope_factor, shape.rope_low_freq,
                            shape.rope_high_freq, shape.rope_orig_max_pos)
        return cls(n_heads=shape.n_heads, n_kv_heads=shape.n_kv_heads, inv_freq=inv,
                   tok=embed["tok"].astype(np.float64), lnf_g=embed["lnf_g"].astype(np.float64),
                   lm_head=embed["lm_head"].astype(np.float64),
                   layers=[layer_from_masters(m, wfmt) for m in layer_masters], s_max=s_max)

    def head(self, h_last: np.ndarray) -> np.ndarray:
        return rms_norm(h_last, self.lnf_g) @ self.lm_head.T

    def forward(self, ids: np.ndarray, all_logits: bool = False) -> np.ndarray:
        ids = np.asarray(ids)
        b, n = ids.shape
        if self.past == 0:
            dkv = self.layers[0].w_qkv.shape[0] - self.tok.shape[1]
            dkv //= 2
            self.kc = [np.zeros((b, self.s_max, dkv)) for _ in self.layers]
            self.vc = [np.zeros((b, self.s_max, dkv)) for _ in self.layers]
        if self.past + n > self.s_max:
            raise ValueError("sequence exceeds s_max")
        h = self.tok[ids]
        self.capture = []
        for j, w in enumerate(self.layers):
            h = decoder_layer(h, w, self.kc[j], self.vc[j], self.past, self.n_heads, self.n_kv_heads, self.inv_freq)
            self.capture.append(h.copy())
        self.past += n
        return self.head(h) if all_logits else self.head(h[:, -1])

    def prefill(self, ids: np.ndarray) -> np.ndarray:
        self.past = 0
        return self.forward(ids)

    def decode(self, ids: np.ndarray) -> np.ndarray:
        return self.forward(np.asarray(ids).reshape(-1, 1))
