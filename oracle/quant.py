"""INT4 group-64 weight quantization — oracle (TEST INFRASTRUCTURE ONLY).

Follows, step by step, the encoding the paper leaves to SPEC.md and that
SURVEY.md §8(c) step 1 fixes (readings Q1/Q2 in DESIGN.md):

  PAPER.md:96 (§2)      "PIPO supports quantizing both weights and KV-cache to INT4"
  PAPER.md:305-309 (§3.4) matrix-vector products "directly on 4-bit quantized weights"
  SPEC.md:459-461        QuantTensor: packed 4-bit codes (two per byte); per-group
                         FP16 scales; group size 64
  SPEC.md:485-493        symmetric per-group scaling; codes in [-8, 7];
                         round-half-to-even; error <= scale/2

For each row n of W[N x K] (K % 64 == 0) and each group g = W[n, 64c:64c+64]:
  a = max|g|                               (fp32)
  s = fp16_rne(a / 7.0f)                   (IEEE fp32 division, then RNE to fp16)
  q = 0                                    if s == 0
  q_k = clamp(rint_rne(g_k / float(s)), -8, 7)   otherwise (fp32 division)
  w_hat_k = float(q_k) * float(s)          (exact in fp32)
Packing: byte k/2 of row n holds q[2m] in bits 0-3 and q[2m+1] in bits 4-7,
two's complement.  Scales: uint16 (fp16 bits) array [N][K/64].
Unpack+scale (kernel K8 contract): fp16_rne(float(q) * float(s)).

Inputs that are non-finite, or whose scale overflows fp16 (|w| > 7*65504), are
outside the encoding's domain and raise ValueError (the library returns
PIPO_E_INVALID_ARG for the same inputs).
"""
from __future__ import annotations

import numpy as np

GROUP = 64
QMIN, QMAX = -8, 7


def quantize_int4_g64(w: np.ndarray):
    """w: float32 [N, K] -> (codes int8 [N, K] in [-8, 7], scales float16 [N, K/64])."""
    w = np.asarray(w)
    if w.dtype != np.float32:
        raise TypeError("quantize_int4_g64 takes float32 masters")
    if w.ndim != 2 or w.shape[1] % GROUP != 0:
        raise ValueError("W must be [N, K] with K % 64 == 0")
    if not np.all(np.isfinite(w)):
        raise ValueError("non-finite weight")
    n, k = w.shape
    g = w.reshape(n, k // GROUP, GROUP)
    a = np.max(np.abs(g), axis=2)                          # fp32
    with np.errstate(over="ignore"):
        s16 = (a / np.float32(7.0)).astype(np.float16)     # fp32 divide, RNE to fp16
    if not np.all(np.isfinite(s16)):
        raise ValueError("group scale overflows fp16")
    s32 = s16.astype(np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.rint(g / s32[:, :, None])                   # fp32 divide, RNE
    q = np.where(s32[:, :, None] == 0, np.float32(0), q)
    q = np.clip(q, QMIN, QMAX).astype(np.int8)
    return q.reshape(n, k), s16


def pack_int4(codes: np.ndarray) -> np.ndarray:
    """codes int8 [N, K] -> packed uint8 [N, K/2] (low nibble = even k)."""
    c = (np.asarray(codes).astype(np.int16) & 0xF).astype(np.uint8)
    return (c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8)


def unpack_int4(packed: np.ndarray) -> np.ndarray:
    """packed uint8 [N, K/2] -> codes int8 [N, K] (two's-complement nibbles)."""
    p = np.asarray(packed, dtype=np.uint8)
    lo = (p & 0xF).astype(np.int16)
    hi = (p >> 4).astype(np.int16)
    lo = np.where(lo >= 8, lo - 16, lo)
    hi = np.where(hi >= 8, hi - 16, hi)
    out = np.empty((p.shape[0], p.shape[1] * 2), dtype=np.int8)
    out[:, 0::2] = lo
    out[:, 1::2] = hi
    return out


def scales_to_bits(s16: np.ndarray) -> np.ndarray:
    return np.asarray(s16, dtype=np.float16).view(np.uint16)


def dequantize(codes: np.ndarray, s16: np.ndarray) -> np.ndarray:
    """w_hat = float(q) * float(s), exact in float32 (<= 4 x 11 significant bits)."""
    n, k = codes.shape
    s = np.repeat(np.asarray(s16, dtype=np.float16).astype(np.float32), GROUP, axis=1)
    return codes.astype(np.float32) * s


def unpack_scale_fp16(packed: np.ndarray, s16: np.ndarray) -> np.ndarray:
    """Kernel K8 contract: fp16_rne(float(q) * float(s)) from packed codes + fp16 scales."""
    return dequantize(unpack_int4(packed), s16).astype(np.float16)


def quant_dequant(w: np.ndarray) -> np.ndarray:
    """The weight the int4 path multiplies by: dequantize(quantize(w)) in float32."""
    q, s = quantize_int4_g64(np.asarray(w, dtype=np.float32))
    return dequantize(q, s)
