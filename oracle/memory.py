"""Memory model and automatic configuration (Eq. 1) — oracle (TEST INFRASTRUCTURE ONLY).

The paper's formulas, written out in exact rational arithmetic (fractions.Fraction)
in the paper's notation, in the order the paper states them:

  PAPER.md:318-331 (§3.5)  l, d, V, p, b, s, h, h_kv; d_h = m * ceil(gamma * floor(8d/3) / m)
                           W = 2 W_embed + l (W_mha + W_mlp); W_embed = p d V;
                           W_mha = p d (2d + d h_kv/h + 1)  [§3.5]  /  p d (2d + 2d h_kv/h + 1)
                           [App. B] -> reading Q23: App. B's form (K and V both scaled);
                           W_mlp = p d (3 d_h + 1);  C = 2 p b s l d h_kv / h
  PAPER.md:498-552 (App. B) M_mha, M_mlp, M_embed for prefill / decode, with / without
                           preloading; M = max of the three.  Reading Q24: where a line's
                           definition and its expansion disagree (decode M_mlp "C/l" vs
                           "4pbsd h_kv/h", decode M_attn "pbh" vs "pb(5d+hs)", decode
                           M_embed "pbsV" vs "pb(d+V)"), the expansion — the last form of
                           each equation — is taken literally; the max(W_mha, W_embed)
                           term is kept un-simplified.
  PAPER.md:339-357 (Eq. 1)  weight tier GPU if W + M < M_GPU; CPU if W + C < M_CPU and
                           B_SSD < B_GPU; else disk.  Pipeline performance-optimized if
                           M < M_GPU else memory-efficient; M = prefill with preloading
                           (PAPER.md:332).  Reading Q25: memory-efficient
                           must still fit the no-preload prefill peak, else infeasible.
  PAPER.md:462-464 (App. A) block size: reading Q26 — the smallest
                           probed size whose min-over-edges throughput is within 5 % of
                           the best.
  PAPER.md:360 (§3.5)      INT4 compute kernel for batch sizes less than 16.

Reading Q27 (OPT): the paper's formulas are written for LLaMA3.1 (three d x d_h MLP
matrices and three d_h-wide intermediates, "3 d_h" / "3 M_w"); for OPT's fc1/fc2 the
factor 3 becomes mlp_mats = 2 with d_h = ffn_dim.

Precision (SPEC.md:133 design decision): p_w for weight terms, p_a for activation and
KV terms ("INT4 precision for weights, with intermediate activations in
FP16").  int4-g64 weights: p_w = 1/2 + 2/64 = 17/32 bytes per element.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction as Fr

P_INT4_G64 = Fr(17, 32)
P_FP16 = Fr(2)


def ffn_hidden_dim(d: int, m: int, gamma: float) -> int:
    """d_h = m * ceil(gamma * floor(8d/3) / m)."""
    return m * math.ceil(gamma * ((8 * d) // 3) / m)


@dataclass(frozen=True)
class Spec:
    l: int
    d: int
    V: int
    h: int
    h_kv: int
    d_h: int
    p_w: Fr = P_FP16
    p_a: Fr = P_FP16
    mlp_mats: int = 3      # 3 = the paper's LLaMA SwiGLU (gate, up, down); 2 = OPT fc1/fc2 (Q27)


def weight_sizes(sp: Spec) -> dict:
    p, d = Fr(sp.p_w), sp.d
    w_embed = p * d * sp.V
    w_mha = p * d * (2 * d + 2 * d * Fr(sp.h_kv, sp.h) + 1)
    w_mlp = p * d * (sp.mlp_mats * sp.d_h + 1)
    return {"w_embed": w_embed, "w_mha": w_mha, "w_mlp": w_mlp,
            "w_total": 2 * w_embed + sp.l * (w_mha + w_mlp)}


def kv_cache_size(sp: Spec, b: int, s: int) -> Fr:
    """C = 2 p b s l d h_kv / h."""
    return 2 * Fr(sp.p_a) * b * s * sp.l * sp.d * Fr(sp.h_kv, sp.h)


def peak_memory(sp: Spec, b: int, s: int, stage: str, preload: bool) -> dict:
    """App. B, expanded forms."""
    W = weight_sizes(sp)
    pa, d, h, V, dh = Fr(sp.p_a), sp.d, sp.h, sp.V, sp.d_h
    mm = sp.mlp_mats
    r = Fr(sp.h_kv, sp.h)
    w_mha, w_mlp, w_embed = W["w_mha"], W["w_mlp"], W["w_embed"]
    if stage == "prefill":
        if preload:
            m_mha = pa * b * s * (5 * d + h * s) + w_mha + w_mlp + 2 * pa * b * s * d * r
            m_mlp = pa * b * s * (mm * dh + 2 * d) + w_mlp + w_mha
            m_embed = pa * b * s * (d + V) + max(w_mha, w_embed) + w_embed
        else:
            m_mha = pa * b * s * (5 * d + h * s) + w_mha + 2 * pa * b * s * d * r
            m_mlp = pa * b * s * (mm * dh + 2 * d) + w_mlp
            m_embed = pa * b * s * (d + V) + w_embed
    elif stage == "decode":
        if preload:
            m_mha = pa * b * (5 * d + h) + w_mha + w_mlp + 4 * pa * b * s * d * r
            m_mlp = pa * b * (mm * dh + 2 * d) + w_mlp + w_mha + 4 * pa * b * s * d * r
            m_embed = pa * b * (d + V) + max(w_mha, w_embed) + w_embed
        else:
            m_mha = pa * b * (5 * d + h * s) + w_mha + 2 * pa * b * s * d * r
            m_mlp = pa * b * (mm * dh + 2 * d) + w_mlp
            m_embed = pa * b * (d + V) + w_embed
    else:
        raise ValueError(stage)
    return {**W, "c_total": kv_cache_size(sp, b, s), "m_mha": m_mha, "m_mlp": m_mlp, "m_embed": m_embed,
            "m_peak": max(m_mha, m_mlp, m_embed)}


def choose_block_size(sizes, h2d, disk=None) -> int:
    """Smallest probed size whose min-over-edges throughput is within 5 % of the best."""
    if not sizes:
        raise ValueError("empty profile")
    eff = [min(a, b) if disk is not None else a for a, b in zip(h2d, disk if disk is not None else h2d)]
    best = max(eff)
    return min(sz for sz, e in zip(sizes, eff) if e >= 0.95 * best)


def choose_plan(sp: Spec, b: int, s: int, M_GPU, M_CPU, B_GPU, B_SSD) -> dict:
    """Eq. (1) as an else-chain."""
    W = weight_sizes(sp)["w_total"]
    C = kv_cache_size(sp, b, s)
    M = peak_memory(sp, b, s, "prefill", True)["m_peak"]
    if W + M < M_GPU:
        tier = "gpu"
    elif W + C < M_CPU and B_SSD < B_GPU:
        tier = "cpu"
    else:
        tier = "disk"
    if M < M_GPU:
        mode = "performance"
    elif peak_memory(sp, b, s, "prefill", False)["m_peak"] < M_GPU:
        mode = "memory_efficient"
    else:
        raise ValueError("infeasible: even the memory-efficient pipeline exceeds M_GPU")
    return {"tier": tier, "mode": mode, "W": W, "C": C, "M": M,
            "use_quant_kernel": sp.p_w < 2 and b < 16}
