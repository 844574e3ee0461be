"""Thin ctypes binding of include/pipo.h — argument marshalling only.

Every function keeps the C-ABI name; all compute happens in libpipo.so (CUDA,
sm_100a).  There is no CPU fallback: importing this module without the built
library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libpipo.so")
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"PIPO CUDA library not built: {_LIB_PATH} missing "
                      "(run __graft_entry__.build() or python -m paper_2504_03664_b200.build)")
_lib = C.CDLL(_LIB_PATH)

PIPO_OK, PIPO_E_INVALID_ARG, PIPO_E_STATE, PIPO_E_OOM, PIPO_E_IO, PIPO_E_FORMAT, PIPO_E_INFEASIBLE, PIPO_E_CUDA = range(8)
STATUS_NAMES = ["OK", "INVALID_ARG", "STATE", "OOM", "IO", "FORMAT", "INFEASIBLE", "CUDA"]
PIPO_W_FP16, PIPO_W_INT4_G64 = 0, 1
PIPO_TIER_DEVICE, PIPO_TIER_HOST, PIPO_TIER_DISK = 0, 1, 2
PIPO_F_TIMELINE = 1
PIPO_F_KPROF = 2
PIPO_F_AUTO_PLAN = 4
K_CLASSES = ["linear_decode", "attn_decode", "lm_head", "linear_prefill", "attn_prefill", "misc"]
PIPO_LAYER_EMBED = -1
PATH_AUTO, PATH_GEMV, PATH_GEMM, PATH_TC, PATH_WS, PATH_TM, PATH_TP, PATH_STREAM, PATH_HEAD, PATH_PAIR = 0, 1, 2, 3, 4, 5, 6, 7, 8, 9

_f = C.POINTER(C.c_float)
_u8 = C.POINTER(C.c_uint8)
_u16 = C.POINTER(C.c_uint16)
_i32 = C.POINTER(C.c_int32)


class pipo_config(C.Structure):
    _fields_ = [("device", C.c_int32), ("d_model", C.c_int32), ("n_layers", C.c_int32), ("n_heads", C.c_int32),
                ("ffn_dim", C.c_int32), ("vocab", C.c_int32), ("max_pos", C.c_int32),
                ("max_batch", C.c_int32), ("max_seq", C.c_int32), ("wfmt", C.c_int32),
                ("weight_tier", C.c_int32), ("kv_tier", C.c_int32), ("kv_fmt", C.c_int32), ("ring_layers", C.c_int32),
                ("chunk_bytes", C.c_int64), ("gemv_max_m", C.c_int32), ("disk_threads", C.c_int32),
                ("disk_dir", C.c_char_p), ("flags", C.c_uint32),
                ("arch", C.c_int32), ("n_kv_heads", C.c_int32), ("rope_theta", C.c_float), ("rope_factor", C.c_float),
                ("rope_low_freq", C.c_float), ("rope_high_freq", C.c_float), ("rope_orig_max_pos", C.c_int32),
                ("numa_node", C.c_int32), ("hbm_budget", C.c_int64)]


PIPO_ARCH_OPT, PIPO_ARCH_LLAMA = 0, 1
PIPO_NUMA_GPU_LOCAL, PIPO_NUMA_NONE = -1, -2


class pipo_layer_weights(C.Structure):
    _fields_ = [(n, _f) for n in ("ln1_g", "ln1_b", "w_qkv", "b_qkv", "w_out", "b_out",
                                  "ln2_g", "ln2_b", "w_fc1", "b_fc1", "w_fc2", "b_fc2")]


class pipo_embed_weights(C.Structure):
    _fields_ = [(n, _f) for n in ("tok", "pos", "lnf_g", "lnf_b", "lm_head")]


class pipo_kstats(C.Structure):
    _fields_ = [("units", C.c_int64), ("ms", C.c_double), ("bytes", C.c_double), ("flops", C.c_double)]


class pipo_stats(C.Structure):
    _fields_ = [("prefill_calls", C.c_int64), ("decode_steps", C.c_int64), ("tokens_generated", C.c_int64),
                ("prefill_s", C.c_double), ("decode_s", C.c_double), ("ttft_s", C.c_double),
                ("decode_tokens_per_s", C.c_double), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("h2d_gbs", C.c_double), ("copy_busy", C.c_double), ("kernel_busy", C.c_double),
                ("union_busy", C.c_double), ("window_s", C.c_double), ("kernel_launches", C.c_int64),
                ("hbm_bytes", C.c_int64), ("pinned_host_bytes", C.c_int64), ("numa_node", C.c_int32),
                ("timeline_truncated", C.c_int32), ("numa_local_frac", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class pipo_mem_spec(C.Structure):
    _fields_ = [("n_layers", C.c_int64), ("d_model", C.c_int64), ("vocab", C.c_int64), ("n_heads", C.c_int64),
                ("n_kv_heads", C.c_int64), ("ffn_hidden", C.c_int64), ("mlp_mats", C.c_int32),
                ("p_weight", C.c_double), ("p_act", C.c_double)]


class pipo_mem_report(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("w_embed", "w_mha", "w_mlp", "w_total", "c_total", "m_mha", "m_mlp",
                                          "m_embed", "m_peak")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class pipo_hw_spec(C.Structure):
    _fields_ = [("m_gpu", C.c_double), ("m_cpu", C.c_double), ("b_gpu", C.c_double), ("b_ssd", C.c_double)]


class pipo_plan(C.Structure):
    _fields_ = [("weight_tier", C.c_int32), ("ring_layers", C.c_int32), ("use_quant_kernel", C.c_int32),
                ("gemv_max_m", C.c_int32), ("block_bytes", C.c_int64), ("w_total", C.c_double),
                ("c_total", C.c_double), ("m_peak", C.c_double), ("m_peak_no_preload", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


PIPO_STAGE_PREFILL, PIPO_STAGE_DECODE = 0, 1


def _sig(name, restype, *args):
    fn = getattr(_lib, name)
    fn.restype = restype
    fn.argtypes = list(args)
    return fn


_P = C.c_void_p
_sig("pipo_last_error", C.c_char_p)
_sig("pipo_abi_version", C.c_int32)
_sig("pipeline_init", C.c_int, C.POINTER(pipo_config), C.POINTER(_P))
_sig("pipeline_destroy", None, _P)
_sig("load_layer_weights", C.c_int, _P, C.c_int32, _P)
_sig("pipo_load_synthetic", C.c_int, _P, C.c_int32, C.c_uint64)
_sig("prefill", C.c_int, _P, _i32, C.c_int32, C.c_int32, _i32, _f)
_sig("decode_step", C.c_int, _P, _i32, _i32, _f)
_sig("decode_step_dev", C.c_int, _P, _P, _P)
_sig("pipeline_stats", C.c_int, _P, C.POINTER(pipo_stats))
_sig("pipeline_stats_reset", C.c_int, _P)
_sig("pipo_set_flags", C.c_int, _P, C.c_uint32)
_sig("pipo_debug_inject", C.c_int, _P, C.c_int32, C.c_int32, C.c_int32)
_sig("pipo_bench_attention_prefill", C.c_int, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
     C.c_int32, C.POINTER(C.c_double))
_sig("pipo_debug_ring_checksums", C.c_int, _P, C.POINTER(C.c_uint64))
_sig("pipo_debug_read_blob", C.c_int, _P, C.c_int32, C.POINTER(C.c_uint8), C.c_int64)
_sig("pipo_layer_blob_bytes", C.c_int, _P, C.POINTER(C.c_int64))
_sig("pipo_stream", _P, _P, C.c_int32)
_sig("pipo_kernel_stats", C.c_int, _P, C.c_int32, C.POINTER(pipo_kstats))
_sig("pipo_quantize_int4_g64", C.c_int, _f, C.c_int64, C.c_int64, _u8, _u16)
_sig("pipo_quantize_int4_g64_gpu", C.c_int, _P, _f, C.c_int64, C.c_int64, _u8, _u16)
_sig("pipo_unpack_int4_g64", C.c_int, _P, _u8, _u16, C.c_int64, C.c_int64, _u16)
_sig("pipo_linear", C.c_int, _P, C.c_int32, C.c_int32, _u16, _f, _f, C.c_int32, C.c_int32, C.c_int32, _f)
_sig("pipo_bench_linear", C.c_int, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
     C.POINTER(C.c_double))
_sig("pipo_probe_bulk", C.c_int, _P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double))
_sig("pipo_bench_attention", C.c_int, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
     C.POINTER(C.c_double))
_sig("pipo_attention_decode", C.c_int, _P, _u16, _u16, _u16, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _f)
_sig("pipo_attention_prefill", C.c_int, _P, _u16, _u16, _u16, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
     C.c_int32, C.c_int32, _f)
_sig("pipo_attention_gqa", C.c_int, _P, _u16, _u16, _u16, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
     C.c_int32, C.c_int32, _f)
_sig("pipo_rope", C.c_int, _P, _u16, _u16, C.c_int32, C.c_int32, C.c_int32, _f, _f)
_sig("pipo_gpu_numa_node", C.c_int32, C.c_int32)
_sig("pipo_probe_disk", C.c_int, C.c_char_p, C.c_int32, C.c_int32, C.c_int64, C.POINTER(C.c_double),
     C.POINTER(C.c_uint64))
_sig("pipo_shard_range", C.c_int, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64))
_sig("pipo_nccl_unique_id", C.c_int, _u8)
_sig("pipo_shard_stream_init", C.c_int, _P, C.c_int32, C.c_int32, _u8)
_sig("pipo_shard_p2p_export", C.c_int, _P, C.c_int32, C.c_int32, _u8)
_sig("pipo_shard_p2p_init", C.c_int, _P, _u8)
_sig("pipo_debug_capture", C.c_int, _P, C.c_int32, _f)
_sig("pipo_probe_h2d", C.c_int, _P, C.c_int64, C.c_int32, C.POINTER(C.c_double))
_sig("pipo_debug_read_rows", C.c_int, _P, C.c_int32, C.c_int32, C.c_int64, C.c_int64, _u8, _u16, _u16)
_sig("pipo_ffn_hidden_dim", C.c_int64, C.c_int64, C.c_int64, C.c_double)
_sig("pipo_memory_model", C.c_int, C.POINTER(pipo_mem_spec), C.c_int64, C.c_int64, C.c_int32, C.c_int32,
     C.POINTER(pipo_mem_report))
_sig("pipo_choose_block_size", C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double),
     C.c_int32)
_sig("pipo_get_plan", C.c_int, _P, C.POINTER(pipo_plan))
_sig("pipo_choose_plan", C.c_int, C.POINTER(pipo_mem_spec), C.c_int64, C.c_int64, C.POINTER(pipo_hw_spec),
     C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32, C.POINTER(pipo_plan))

EXPORTED = ["pipo_last_error", "pipo_abi_version", "pipeline_init", "pipeline_destroy", "load_layer_weights",
            "pipo_load_synthetic", "prefill", "decode_step", "decode_step_dev", "pipeline_stats",
            "pipeline_stats_reset", "pipo_stream", "pipo_kernel_stats", "pipo_quantize_int4_g64", "pipo_quantize_int4_g64_gpu",
            "pipo_unpack_int4_g64", "pipo_linear", "pipo_bench_linear", "pipo_probe_bulk", "pipo_bench_attention", "pipo_attention_decode", "pipo_attention_prefill", "pipo_debug_capture", "pipo_probe_h2d", "pipo_debug_read_rows",
            "pipo_attention_gqa", "pipo_rope", "pipo_set_flags", "pipo_debug_inject", "pipo_debug_ring_checksums", "pipo_bench_attention_prefill",
            "pipo_debug_read_blob", "pipo_layer_blob_bytes", "pipo_shard_range", "pipo_gpu_numa_node", "pipo_nccl_unique_id", "pipo_shard_stream_init", "pipo_shard_p2p_export", "pipo_shard_p2p_init",
            "pipo_ffn_hidden_dim", "pipo_probe_disk", "pipo_memory_model", "pipo_choose_block_size", "pipo_choose_plan", "pipo_get_plan"]


class PipoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


def _check(st):
    if st != PIPO_OK:
        raise PipoError(st, _lib.pipo_last_error().decode(errors="replace"))


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def lib_path():
    return _LIB_PATH


def pipo_abi_version():
    return _lib.pipo_abi_version()


def pipeline_init(cfg: pipo_config):
    h = _P()
    _check(_lib.pipeline_init(C.byref(cfg), C.byref(h)))
    return h


def pipeline_destroy(ctx):
    _lib.pipeline_destroy(ctx)


def load_layer_weights(ctx, layer: int, w: dict):
    if layer == PIPO_LAYER_EMBED:
        # absent tensors (LLaMA: pos, lnf_b; OPT: lm_head) are passed as NULL
        keep = {k: _c(w[k], np.float32) for k in ("tok", "pos", "lnf_g", "lnf_b", "lm_head") if w.get(k) is not None}
        st = pipo_embed_weights(**{k: _ptr(v, C.c_float) for k, v in keep.items()})
    else:
        names = [n for n, _ in pipo_layer_weights._fields_]
        keep = {k: _c(w[k], np.float32) for k in names if w.get(k) is not None}   # LLaMA: no biases
        st = pipo_layer_weights(**{k: _ptr(v, C.c_float) for k, v in keep.items()})
    _check(_lib.load_layer_weights(ctx, layer, C.byref(st)))


def pipo_load_synthetic(ctx, layer: int, seed: int):
    _check(_lib.pipo_load_synthetic(ctx, layer, seed))


def prefill(ctx, tokens, want_logits=False, vocab=None):
    t = _c(tokens, np.int32)
    b, p = t.shape
    nxt = np.empty(b, dtype=np.int32)
    lg = np.empty((b, vocab), dtype=np.float32) if want_logits else None
    _check(_lib.prefill(ctx, _ptr(t, C.c_int32), b, p, _ptr(nxt, C.c_int32),
                        _ptr(lg, C.c_float) if lg is not None else None))
    return nxt, lg


def decode_step(ctx, tokens, want_logits=False, vocab=None):
    t = _c(tokens, np.int32)
    nxt = np.empty(t.shape[0], dtype=np.int32)
    lg = np.empty((t.shape[0], vocab), dtype=np.float32) if want_logits else None
    _check(_lib.decode_step(ctx, _ptr(t, C.c_int32), _ptr(nxt, C.c_int32),
                            _ptr(lg, C.c_float) if lg is not None else None))
    return nxt, lg


def decode_step_dev(ctx, tokens_dev_ptr: int, next_dev_ptr: int):
    _check(_lib.decode_step_dev(ctx, C.c_void_p(tokens_dev_ptr), C.c_void_p(next_dev_ptr)))


def pipeline_stats(ctx) -> dict:
    s = pipo_stats()
    _check(_lib.pipeline_stats(ctx, C.byref(s)))
    return s.as_dict()


def pipeline_stats_reset(ctx):
    _check(_lib.pipeline_stats_reset(ctx))


def pipo_kernel_stats(ctx) -> dict:
    out = {}
    for i, name in enumerate(K_CLASSES):
        k = pipo_kstats()
        _check(_lib.pipo_kernel_stats(ctx, i, C.byref(k)))
        out[name] = {"units": k.units, "ms": k.ms, "bytes": k.bytes, "flops": k.flops}
    return out


def pipo_stream(ctx, which=0) -> int:
    return _lib.pipo_stream(ctx, which) or 0


def pipo_quantize_int4_g64(w):
    w = _c(w, np.float32)
    rows, cols = w.shape
    codes = np.empty((rows, cols // 2), dtype=np.uint8)
    scales = np.empty((rows, cols // 64), dtype=np.uint16)
    _check(_lib.pipo_quantize_int4_g64(_ptr(w, C.c_float), rows, cols, _ptr(codes, C.c_uint8),
                                       _ptr(scales, C.c_uint16)))
    return codes, scales


def pipo_quantize_int4_g64_gpu(ctx, w):
    w = _c(w, np.float32)
    rows, cols = w.shape
    codes = np.empty((rows, cols // 2), dtype=np.uint8)
    scales = np.empty((rows, cols // 64), dtype=np.uint16)
    _check(_lib.pipo_quantize_int4_g64_gpu(ctx, _ptr(w, C.c_float), rows, cols, _ptr(codes, C.c_uint8),
                                           _ptr(scales, C.c_uint16)))
    return codes, scales


def pipo_unpack_int4_g64(ctx, codes, scales):
    codes = _c(codes, np.uint8)
    scales = _c(scales, np.uint16)
    rows, half = codes.shape
    out = np.empty((rows, half * 2), dtype=np.uint16)
    _check(_lib.pipo_unpack_int4_g64(ctx, _ptr(codes, C.c_uint8), _ptr(scales, C.c_uint16), rows, half * 2,
                                     _ptr(out, C.c_uint16)))
    return out.view(np.float16)


def pipo_linear(ctx, wfmt, path, x, w, bias=None):
    x = _c(np.asarray(x, dtype=np.float16).view(np.uint16), np.uint16)
    w = _c(w, np.float32)
    M, K = x.shape
    N = w.shape[0]
    b = _c(bias, np.float32) if bias is not None else None
    y = np.empty((M, N), dtype=np.float32)
    _check(_lib.pipo_linear(ctx, wfmt, path, _ptr(x, C.c_uint16), _ptr(w, C.c_float),
                            _ptr(b, C.c_float) if b is not None else None, M, N, K, _ptr(y, C.c_float)))
    return y


def pipo_bench_linear(ctx, wfmt, path, M, N, K, iters=20) -> float:
    us = C.c_double()
    _check(_lib.pipo_bench_linear(ctx, wfmt, path, M, N, K, iters, C.byref(us)))
    return us.value


def pipo_probe_bulk(ctx, chunk: int, stages: int, streams: int = 1) -> float:
    g = C.c_double()
    _check(_lib.pipo_probe_bulk(ctx, chunk, stages, streams, C.byref(g)))
    return g.value


def pipo_bench_attention(ctx, b, L, d, n_heads, variant=0, iters=10, n_kv_heads=0) -> float:
    us = C.c_double()
    _check(_lib.pipo_bench_attention(ctx, b, L, d, n_heads, n_kv_heads, variant, iters, C.byref(us)))
    return us.value


def pipo_attention_decode(ctx, q, k, v, n_heads, variant=0):
    q = _c(np.asarray(q, dtype=np.float16).view(np.uint16), np.uint16)
    k = _c(np.asarray(k, dtype=np.float16).view(np.uint16), np.uint16)
    v = _c(np.asarray(v, dtype=np.float16).view(np.uint16), np.uint16)
    b, d = q.shape
    L = k.shape[0]
    o = np.empty((b, d), dtype=np.float32)
    _check(_lib.pipo_attention_decode(ctx, _ptr(q, C.c_uint16), _ptr(k, C.c_uint16), _ptr(v, C.c_uint16),
                                      b, L, d, n_heads, variant, _ptr(o, C.c_float)))
    return o


def pipo_attention_prefill(ctx, q, k, v, past, n_heads, cuda_cores=False):
    q = _c(np.asarray(q, dtype=np.float16).view(np.uint16), np.uint16)
    k = _c(np.asarray(k, dtype=np.float16).view(np.uint16), np.uint16)
    v = _c(np.asarray(v, dtype=np.float16).view(np.uint16), np.uint16)
    b, n, d = q.shape
    o = np.empty((b, n, d), dtype=np.float32)
    _check(_lib.pipo_attention_prefill(ctx, _ptr(q, C.c_uint16), _ptr(k, C.c_uint16), _ptr(v, C.c_uint16),
                                       b, n, past, d, n_heads, int(cuda_cores), _ptr(o, C.c_float)))
    return o


def pipo_attention_gqa(ctx, q, k, v, past, n_heads, n_kv_heads, variant=0):
    """q [b][n][h*hd], k/v [past+n][b][h_kv*hd] (fp16 values) -> o [b][n][h*hd] fp32."""
    q = _c(np.asarray(q, dtype=np.float16).view(np.uint16), np.uint16)
    k = _c(np.asarray(k, dtype=np.float16).view(np.uint16), np.uint16)
    v = _c(np.asarray(v, dtype=np.float16).view(np.uint16), np.uint16)
    b, n, d = q.shape
    o = np.empty((b, n, d), dtype=np.float32)
    _check(_lib.pipo_attention_gqa(ctx, _ptr(q, C.c_uint16), _ptr(k, C.c_uint16), _ptr(v, C.c_uint16), b, n, past,
                                   n_heads, n_kv_heads, d // n_heads, variant, _ptr(o, C.c_float)))
    return o


def pipo_rope(ctx, q, k, past):
    """q [b][n][h*hd], k [past+n][b][h_kv*hd] (fp16 values) -> (q_rot, k_rot) fp32."""
    q = _c(np.asarray(q, dtype=np.float16).view(np.uint16), np.uint16)
    k = _c(np.asarray(k, dtype=np.float16).view(np.uint16), np.uint16)
    b, n, _ = q.shape
    qo = np.empty(q.shape, dtype=np.float32)
    ko = np.empty(k.shape, dtype=np.float32)
    _check(_lib.pipo_rope(ctx, _ptr(q, C.c_uint16), _ptr(k, C.c_uint16), b, n, past, _ptr(qo, C.c_float),
                          _ptr(ko, C.c_float)))
    return qo, ko


def pipo_gpu_numa_node(device: int) -> int:
    return _lib.pipo_gpu_numa_node(device)


def pipo_shard_range(layer_bytes: int, world: int, rank: int):
    """(offset, bytes) of rank's range of a padded layer blob (host-only, NEXT-1)."""
    off, n = C.c_int64(), C.c_int64()
    _check(_lib.pipo_shard_range(layer_bytes, world, rank, C.byref(off), C.byref(n)))
    return off.value, n.value


def pipo_nccl_unique_id() -> bytes:
    buf = np.zeros(128, dtype=np.uint8)
    _check(_lib.pipo_nccl_unique_id(_ptr(buf, C.c_uint8)))
    return buf.tobytes()


def pipo_shard_stream_init(ctx, rank: int, world: int, uid: bytes):
    buf = np.frombuffer(uid, dtype=np.uint8).copy()
    assert buf.size == 128
    _check(_lib.pipo_shard_stream_init(ctx, rank, world, _ptr(buf, C.c_uint8)))


PIPO_SHARD_HANDLE_BYTES = 128


def pipo_shard_p2p_export(ctx, rank: int, world: int) -> bytes:
    buf = np.zeros(PIPO_SHARD_HANDLE_BYTES, dtype=np.uint8)
    _check(_lib.pipo_shard_p2p_export(ctx, rank, world, _ptr(buf, C.c_uint8)))
    return buf.tobytes()


def pipo_shard_p2p_init(ctx, handles: list):
    """handles: every rank's export blob, in rank order."""
    buf = np.frombuffer(b"".join(handles), dtype=np.uint8).copy()
    assert buf.size == PIPO_SHARD_HANDLE_BYTES * len(handles)
    _check(_lib.pipo_shard_p2p_init(ctx, _ptr(buf, C.c_uint8)))


def pipo_set_flags(ctx, flags: int):
    _check(_lib.pipo_set_flags(ctx, flags))


def pipo_bench_attention_prefill(ctx, b, n, d, n_heads, variant=0, iters=5, n_kv_heads=0) -> float:
    us = C.c_double()
    _check(_lib.pipo_bench_attention_prefill(ctx, b, n, d, n_heads, n_kv_heads, variant, iters, C.byref(us)))
    return us.value


def pipo_debug_inject(ctx, copy_delay_us: int = 0, compute_delay_us: int = 0, ring_checksum: bool = False):
    _check(_lib.pipo_debug_inject(ctx, copy_delay_us, compute_delay_us, 1 if ring_checksum else 0))


def pipo_debug_ring_checksums(ctx, n_layers: int) -> np.ndarray:
    out = np.zeros(n_layers, np.uint64)
    _check(_lib.pipo_debug_ring_checksums(ctx, out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out


def pipo_debug_read_blob(ctx, layer: int) -> np.ndarray:
    n = C.c_int64()
    _check(_lib.pipo_layer_blob_bytes(ctx, C.byref(n)))
    out = np.zeros(n.value, np.uint8)
    _check(_lib.pipo_debug_read_blob(ctx, layer, out.ctypes.data_as(C.POINTER(C.c_uint8)), n.value))
    return out


def pipo_debug_capture(ctx, out: np.ndarray | None):
    if out is None:
        _check(_lib.pipo_debug_capture(ctx, 0, None))
    else:
        assert out.dtype == np.float32 and out.flags.c_contiguous
        _check(_lib.pipo_debug_capture(ctx, 1, _ptr(out, C.c_float)))


def pipo_debug_read_rows(ctx, layer: int, matrix: int, row0: int, nrows: int, K: int, int4: bool):
    """Stored rows in canonical form: int4 -> (codes [nrows][K/2] u8, scales [nrows][K/64] fp16 bits);
    fp16 / embeddings -> values [nrows][K] float16."""
    if int4:
        codes = np.empty((nrows, K // 2), dtype=np.uint8)
        scales = np.empty((nrows, K // 64), dtype=np.uint16)
        _check(_lib.pipo_debug_read_rows(ctx, layer, matrix, row0, nrows, _ptr(codes, C.c_uint8),
                                         _ptr(scales, C.c_uint16), None))
        return codes, scales
    vals = np.empty((nrows, K), dtype=np.uint16)
    _check(_lib.pipo_debug_read_rows(ctx, layer, matrix, row0, nrows, None, None, _ptr(vals, C.c_uint16)))
    return vals.view(np.float16)


def pipo_probe_h2d(ctx, nbytes: int, reps: int = 5) -> float:
    g = C.c_double()
    _check(_lib.pipo_probe_h2d(ctx, nbytes, reps, C.byref(g)))
    return g.value


def pipo_probe_disk(directory: str, n_layers: int, threads: int = 4, chunk: int = 32 << 20,
                    checksum: bool = False):
    """Disk-tier roofline probe (no GPU): (GB/s, checksum or None)."""
    g = C.c_double()
    cs = C.c_uint64()
    _check(_lib.pipo_probe_disk(str(directory).encode(), n_layers, threads, chunk, C.byref(g),
                                C.byref(cs) if checksum else None))
    return g.value, (cs.value if checksum else None)


def mem_spec(*, l, d, V, h, h_kv, d_h, mlp_mats=3, p_weight=2.0, p_act=2.0) -> pipo_mem_spec:
    """pipo_mem_spec in the paper's notation."""
    return pipo_mem_spec(n_layers=l, d_model=d, vocab=V, n_heads=h, n_kv_heads=h_kv, ffn_hidden=d_h,
                         mlp_mats=mlp_mats, p_weight=float(p_weight), p_act=float(p_act))


def pipo_ffn_hidden_dim(d: int, m: int, gamma: float) -> int:
    return _lib.pipo_ffn_hidden_dim(d, m, gamma)


def pipo_memory_model(spec: pipo_mem_spec, b: int, s: int, stage: int, preload: bool) -> dict:
    r = pipo_mem_report()
    _check(_lib.pipo_memory_model(C.byref(spec), b, s, stage, int(preload), C.byref(r)))
    return r.as_dict()


def _dbl(a):
    return (C.c_double * len(a))(*a) if a is not None else None


def pipo_choose_block_size(sizes, h2d_bps, disk_bps=None) -> int:
    n = len(sizes)
    return _lib.pipo_choose_block_size((C.c_int64 * n)(*sizes), _dbl(h2d_bps), _dbl(disk_bps), n)


def pipo_choose_plan(spec: pipo_mem_spec, b: int, s: int, *, m_gpu, m_cpu, b_gpu, b_ssd,
                     sizes=(), h2d_bps=None, disk_bps=None) -> dict:
    hw = pipo_hw_spec(m_gpu=float(m_gpu), m_cpu=float(m_cpu), b_gpu=float(b_gpu), b_ssd=float(b_ssd))
    out = pipo_plan()
    n = len(sizes)
    _check(_lib.pipo_choose_plan(C.byref(spec), b, s, C.byref(hw), (C.c_int64 * n)(*sizes) if n else None,
                                 _dbl(h2d_bps) if n else None, _dbl(disk_bps) if n else None, n, C.byref(out)))
    return out.as_dict()


def pipo_get_plan(ctx) -> dict:
    out = pipo_plan()
    _check(_lib.pipo_get_plan(ctx, C.byref(out)))
    return out.as_dict()


def make_config(shape, *, device=0, max_batch, max_seq, wfmt=PIPO_W_INT4_G64, weight_tier=PIPO_TIER_HOST,
                kv_tier=PIPO_TIER_DEVICE, kv_fmt=PIPO_W_FP16, ring_layers=2, chunk_bytes=0, gemv_max_m=15, disk_threads=4,
                disk_dir=None, flags=PIPO_F_TIMELINE, n_layers=None, numa_node=PIPO_NUMA_GPU_LOCAL,
                hbm_budget=0) -> pipo_config:
    """pipo_config from a pipo_synth.OPTShape-like object (d_model, n_layers, n_heads, ffn_dim, vocab, max_pos)
    or a pipo_synth.LlamaShape (adds n_kv_heads and the llama3 RoPE parameters -> arch LLAMA)."""
    llama = hasattr(shape, "n_kv_heads")
    extra = dict(arch=PIPO_ARCH_LLAMA, n_kv_heads=shape.n_kv_heads, rope_theta=shape.rope_theta,
                 rope_factor=shape.rope_factor, rope_low_freq=shape.rope_low_freq, rope_high_freq=shape.rope_high_freq,
                 rope_orig_max_pos=shape.rope_orig_max_pos) if llama else dict(arch=PIPO_ARCH_OPT)
    return pipo_config(device=device, d_model=shape.d_model, n_layers=n_layers or shape.n_layers,
                       n_heads=shape.n_heads, ffn_dim=shape.ffn_dim, vocab=shape.vocab, max_pos=shape.max_pos,
                       max_batch=max_batch, max_seq=max_seq, wfmt=wfmt, weight_tier=weight_tier, kv_tier=kv_tier,
                       kv_fmt=kv_fmt,
                       ring_layers=ring_layers, chunk_bytes=chunk_bytes, gemv_max_m=gemv_max_m,
                       disk_threads=disk_threads, disk_dir=(disk_dir.encode() if disk_dir else None), flags=flags,
                       numa_node=numa_node, hbm_budget=hbm_budget, **extra)


class Pipeline:
    """Owns one pipo_ctx (one GPU).  Marshalling only."""

    def __init__(self, cfg: pipo_config):
        self.cfg = cfg
        self.vocab = cfg.vocab
        self.ctx = pipeline_init(cfg)

    def close(self):
        if self.ctx:
            pipeline_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_layer_weights(self, layer, w):
        load_layer_weights(self.ctx, layer, w)

    def load_synthetic(self, layer, seed):
        pipo_load_synthetic(self.ctx, layer, seed)

    def prefill(self, tokens, want_logits=False):
        return prefill(self.ctx, tokens, want_logits, self.vocab)

    def decode_step(self, tokens, want_logits=False):
        return decode_step(self.ctx, tokens, want_logits, self.vocab)

    def stats(self):
        return pipeline_stats(self.ctx)

    def stats_reset(self):
        pipeline_stats_reset(self.ctx)
