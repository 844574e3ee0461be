"""Seeded synthetic inputs shared by the oracle side and the GPU side of the tests.

This module holds NONE of the method's arithmetic (no quantization, no layer
math).  It only draws the synthetic OPT weights and prompts described in
DESIGN.md §"Input recipe": every value is a pure function of
(seed, layer slot, tensor id, element index), built from the splitmix64 finalizer
so that the CUDA library (`paper_2504_03664_b200/csrc/synth.cu`) can implement
the *same* counter-based generator independently and produce bit-identical
masters on the GPU (the task's rule: "each side implements the same
counter-based generator").

Distributions ([ext] OPT init_std=0.02):
  * linear weights, token/position embeddings: Irwin-Hall(4) approximation of
    N(0, 0.02): sum of the four 16-bit fields of the hash, centred and scaled
    by one fp32 multiply;
  * biases: U(-0.02, 0.02); LN beta: U(-0.1, 0.1); LN gamma: 1 + U(-0.1, 0.1);
  * prompts: ids uniform in [4, V) (avoids pad=1, bos/eos=2).
Every float master is rounded to fp16 (RNE) and returned as float32, so it is
exactly representable in the fp16 weight formats.

Bit-level recipe (mirrored in csrc/synth.cu):
  mix64(z): z=(z^(z>>30))*0xBF58476D1CE4E5B9; z=(z^(z>>27))*0x94D049BB133111EB; z^(z>>31)
  key(seed, slot, tid) = mix64(mix64(seed) ^ (slot << 16) ^ tid)
  h(i) = mix64(key + (i+1) * 0x9E3779B97F4A7C15)            (all mod 2^64)
  normal(i)  = f16( f32(sum16x4(h) - 131070) * f32(std / sqrt((65536^2-1)/3)) )
  uniform(i) = f16( f32((h >> 40) - 2^23) * f32(a / 2^23) )
  gamma(i)   = f16( 1.0f + f32((h >> 40) - 2^23) * f32(0.1 / 2^23) )   (mul, then add; no FMA)
  token(i)   = 4 + h mod (V - 4)
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)

WEIGHT_SEED = 2504   # SURVEY.md §8(d) "Seeds: weights 2504"
PROMPT_SEED = 3664   # "prompts 3664"

# tensor ids inside a decoder-layer slot (slot = layer + 1)
T_LN1_G, T_LN1_B, T_W_QKV, T_B_QKV, T_W_OUT, T_B_OUT = 0, 1, 2, 3, 4, 5
T_LN2_G, T_LN2_B, T_W_FC1, T_B_FC1, T_W_FC2, T_B_FC2 = 6, 7, 8, 9, 10, 11
# tensor ids inside the embedding slot (slot = 0)
T_TOK, T_POS, T_LNF_G, T_LNF_B = 0, 1, 2, 3
PROMPT_SLOT = 0xFFFF

KIND_NORMAL, KIND_UNIFORM, KIND_GAMMA = 0, 1, 2
W_STD = 0.02
BIAS_A = 0.02
LN_A = 0.1

_N_THREADS = max(1, min(16, len(os.sched_getaffinity(0))))


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * C1
    z = (z ^ (z >> np.uint64(27))) * C2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, slot: int, tid: int) -> np.uint64:
    with np.errstate(over="ignore"):
        s = _mix64(np.array([seed], dtype=np.uint64))[0]
        k = s ^ (np.uint64(slot) << np.uint64(16)) ^ np.uint64(tid)
        return _mix64(np.array([k], dtype=np.uint64))[0]


def _hash(key: np.uint64, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return _mix64(key + (idx.astype(np.uint64) + np.uint64(1)) * GOLDEN)


def normal_scale(std: float) -> np.float32:
    return np.float32(std / np.sqrt((65536.0 * 65536.0 - 1.0) / 3.0))


def uniform_scale(a: float) -> np.float32:
    return np.float32(a / float(1 << 23))


def _values(kind: int, param: float, h: np.ndarray) -> np.ndarray:
    if kind == KIND_NORMAL:
        m = np.uint64(0xFFFF)
        s = (h & m) + ((h >> np.uint64(16)) & m) + ((h >> np.uint64(32)) & m) + (h >> np.uint64(48))
        c = (s.astype(np.int64) - 131070).astype(np.float32)
        v = c * normal_scale(param)
    else:
        c = ((h >> np.uint64(40)).astype(np.int64) - (1 << 23)).astype(np.float32)
        v = c * uniform_scale(param)
        if kind == KIND_GAMMA:
            v = np.float32(1.0) + v
    return v.astype(np.float32).astype(np.float16).astype(np.float32)


def draw(seed: int, slot: int, tid: int, kind: int, param: float, start: int, count: int) -> np.ndarray:
    """Elements [start, start+count) of one tensor stream, as fp16-exact float32."""
    key = stream_key(seed, slot, tid)
    out = np.empty(count, dtype=np.float32)
    chunk = 1 << 20
    spans = [(o, min(chunk, count - o)) for o in range(0, count, chunk)]

    def work(span):
        o, n = span
        idx = np.arange(start + o, start + o + n, dtype=np.uint64)
        out[o:o + n] = _values(kind, param, _hash(key, idx))

    if len(spans) > 1:
        with ThreadPoolExecutor(_N_THREADS) as ex:
            list(ex.map(work, spans))
    elif spans:
        work(spans[0])
    return out


def draw_rows(seed: int, slot: int, tid: int, kind: int, param: float, cols: int, rows) -> np.ndarray:
    """Selected rows of a row-major [*, cols] tensor stream (index = row*cols + col)."""
    rows = np.asarray(rows, dtype=np.int64)
    out = np.empty((len(rows), cols), dtype=np.float32)
    for i, r in enumerate(rows):
        out[i] = draw(seed, slot, tid, kind, param, int(r) * cols, cols)
    return out


@dataclass(frozen=True)
class OPTShape:
    """OPT decoder shape (SURVEY.md §8 'OPT shapes' table; [ext] public OPT configs)."""
    d_model: int
    n_layers: int
    n_heads: int
    ffn_dim: int
    vocab: int = 50272
    max_pos: int = 2048

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads


OPT_125M = OPTShape(768, 12, 12, 3072)
OPT_1_3B = OPTShape(2048, 24, 32, 8192)
OPT_6_7B = OPTShape(4096, 32, 32, 16384)
OPT_13B = OPTShape(5120, 40, 40, 20480)
OPT_30B = OPTShape(7168, 48, 56, 28672)

# (tid, kind, param, shape-fn) for each decoder-layer tensor
def layer_tensor_specs(s: OPTShape):
    d, f = s.d_model, s.ffn_dim
    return {
        "ln1_g": (T_LN1_G, KIND_GAMMA, LN_A, (d,)),
        "ln1_b": (T_LN1_B, KIND_UNIFORM, LN_A, (d,)),
        "w_qkv": (T_W_QKV, KIND_NORMAL, W_STD, (3 * d, d)),
        "b_qkv": (T_B_QKV, KIND_UNIFORM, BIAS_A, (3 * d,)),
        "w_out": (T_W_OUT, KIND_NORMAL, W_STD, (d, d)),
        "b_out": (T_B_OUT, KIND_UNIFORM, BIAS_A, (d,)),
        "ln2_g": (T_LN2_G, KIND_GAMMA, LN_A, (d,)),
        "ln2_b": (T_LN2_B, KIND_UNIFORM, LN_A, (d,)),
        "w_fc1": (T_W_FC1, KIND_NORMAL, W_STD, (f, d)),
        "b_fc1": (T_B_FC1, KIND_UNIFORM, BIAS_A, (f,)),
        "w_fc2": (T_W_FC2, KIND_NORMAL, W_STD, (d, f)),
        "b_fc2": (T_B_FC2, KIND_UNIFORM, BIAS_A, (d,)),
    }


def embed_tensor_specs(s: OPTShape):
    d = s.d_model
    return {
        "tok": (T_TOK, KIND_NORMAL, W_STD, (s.vocab, d)),
        "pos": (T_POS, KIND_NORMAL, W_STD, (s.max_pos + 2, d)),
        "lnf_g": (T_LNF_G, KIND_GAMMA, LN_A, (d,)),
        "lnf_b": (T_LNF_B, KIND_UNIFORM, LN_A, (d,)),
    }


def _draw_spec(seed, slot, spec):
    tid, kind, param, shape = spec
    n = int(np.prod(shape))
    return draw(seed, slot, tid, kind, param, 0, n).reshape(shape)


def layer_masters(s: OPTShape, layer: int, seed: int = WEIGHT_SEED) -> dict:
    """fp32 (fp16-exact) master tensors of decoder layer `layer` (0-based)."""
    return {k: _draw_spec(seed, layer + 1, v) for k, v in layer_tensor_specs(s).items()}


def embed_masters(s: OPTShape, seed: int = WEIGHT_SEED) -> dict:
    return {k: _draw_spec(seed, 0, v) for k, v in embed_tensor_specs(s).items()}


def prompts(b: int, p: int, vocab: int, seed: int = PROMPT_SEED) -> np.ndarray:
    """[b, p] int32 token ids uniform in [4, vocab)."""
    key = stream_key(seed, PROMPT_SLOT, 0)
    h = _hash(key, np.arange(b * p, dtype=np.uint64))
    ids = np.uint64(4) + h % np.uint64(vocab - 4)
    return ids.astype(np.int32).reshape(b, p)


# ---------------------------------------------------------------------------------
# LLaMA3.1-shaped models (NEXT-4; PAPER.md:318-331 §3.5, :390 §4.1).
# Same generator and distributions ([ext] LlamaConfig initializer_range = 0.02; RMSNorm
# weights drawn like LN gamma); tensor ids reuse the OPT slots where the role matches.
T_LM_HEAD = 4   # embedding slot: untied LM head [V][d]


@dataclass(frozen=True)
class LlamaShape:
    """LLaMA3.1 decoder shape ([ext] public Llama-3.1 configs): GQA with n_kv_heads,
    SwiGLU MLP of width ffn_dim (= d_h), RoPE (llama3 frequency rule),
    RMSNorm, untied LM head, no biases."""
    d_model: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    ffn_dim: int
    vocab: int = 128256
    max_pos: int = 131072
    rope_theta: float = 500000.0
    rope_factor: float = 8.0          # llama3 rope_scaling (0 -> plain RoPE)
    rope_low_freq: float = 1.0
    rope_high_freq: float = 4.0
    rope_orig_max_pos: int = 8192

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    @property
    def d_kv(self) -> int:
        return self.n_kv_heads * self.head_dim


LLAMA31_8B = LlamaShape(4096, 32, 32, 8, 14336)
# [ext] Llama-3.2-1B config: rope factor 32 (the paper's offloading-overhead table, PAPER.md:727-742;
# its tied LM head is drawn here as a separate tensor — throughput is unaffected)
LLAMA32_1B = LlamaShape(2048, 16, 32, 8, 8192, rope_factor=32.0)


def llama_layer_tensor_specs(s: LlamaShape):
    d, f, dkv = s.d_model, s.ffn_dim, s.d_kv
    return {
        "ln1_g": (T_LN1_G, KIND_GAMMA, LN_A, (d,)),
        "w_qkv": (T_W_QKV, KIND_NORMAL, W_STD, (d + 2 * dkv, d)),   # rows q | k | v
        "w_out": (T_W_OUT, KIND_NORMAL, W_STD, (d, d)),
        "ln2_g": (T_LN2_G, KIND_GAMMA, LN_A, (d,)),
        "w_fc1": (T_W_FC1, KIND_NORMAL, W_STD, (2 * f, d)),         # rows gate | up
        "w_fc2": (T_W_FC2, KIND_NORMAL, W_STD, (d, f)),             # down
    }


def llama_embed_tensor_specs(s: LlamaShape):
    d = s.d_model
    return {
        "tok": (T_TOK, KIND_NORMAL, W_STD, (s.vocab, d)),
        "lnf_g": (T_LNF_G, KIND_GAMMA, LN_A, (d,)),
        "lm_head": (T_LM_HEAD, KIND_NORMAL, W_STD, (s.vocab, d)),
    }


def llama_layer_masters(s: LlamaShape, layer: int, seed: int = WEIGHT_SEED) -> dict:
    return {k: _draw_spec(seed, layer + 1, v) for k, v in llama_layer_tensor_specs(s).items()}


def llama_embed_masters(s: LlamaShape, seed: int = WEIGHT_SEED) -> dict:
    return {k: _draw_spec(seed, 0, v) for k, v in llama_embed_tensor_specs(s).items()}
