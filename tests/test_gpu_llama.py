"""GPU parity of the LLaMA3.1-shaped path (NEXT-4) vs oracle/llama.py, through the C-ABI.

* kernels: RoPE (llama3 frequencies, q and the fresh K rows of the cache) and GQA
  attention (decode and causal prefill, query head j -> KV head j / group) against the
  oracle's fp64 definitions on the same fp16 inputs;
* whole model, tiny GQA shape (h = 8, h_kv = 2, hd = 64 and 128): every layer output
  (debug capture) and every step's logits within 2e-2 of the fp64 oracle, int4 and fp16
  weights, GEMV (b <= 15) and tensor-core (b >= 16) linear paths, teacher-forced ids;
* the GPU generator + quantizer (pipo_load_synthetic, incl. the tile-interleaved
  gate|up matrix) reproduce the numpy masters + host quantizer bit for bit;
* the method's invariance: DEVICE vs HOST weight tier, ring depth, host-resident KV ->
  bit-identical logits.
"""
import numpy as np
import pytest

import pipo_synth as synth
from oracle import llama
from tests.gpu_util import load_masters, pipo_mod, rel_inf

pytestmark = pytest.mark.gpu

TINY = synth.LlamaShape(d_model=512, n_layers=2, n_heads=8, n_kv_heads=2, ffn_dim=1408, vocab=1000, max_pos=4096,
                        rope_orig_max_pos=64)
TINY128 = synth.LlamaShape(d_model=1024, n_layers=2, n_heads=8, n_kv_heads=4, ffn_dim=2816, vocab=768, max_pos=4096,
                           rope_orig_max_pos=64)


def _masters(shape):
    return synth.llama_embed_masters(shape), [synth.llama_layer_masters(shape, j) for j in range(shape.n_layers)]


@pytest.fixture(scope="module")
def tiny():
    return _masters(TINY)


def test_rope_kernel_vs_oracle():
    pipo = pipo_mod()
    rng = np.random.default_rng(5)
    b, n, past = 3, 5, 7
    s = TINY
    cfg = pipo.make_config(s, max_batch=b, max_seq=past + n + 1, weight_tier=pipo.PIPO_TIER_DEVICE)
    with pipo.Pipeline(cfg) as pl:
        q = rng.standard_normal((b, n, s.d_model)).astype(np.float16)
        k = rng.standard_normal((past + n, b, s.d_kv)).astype(np.float16)
        qo, ko = pipo.pipo_rope(pl.ctx, q, k, past)
    inv = llama.rope_inv_freq(s.head_dim, s.rope_theta, s.rope_factor, s.rope_low_freq, s.rope_high_freq,
                              s.rope_orig_max_pos)
    pos = past + np.arange(n)
    qr = llama.rope(q.astype(np.float64).reshape(b, n, s.n_heads, s.head_dim), pos, inv).reshape(b, n, -1)
    kn = k[past:].astype(np.float64).transpose(1, 0, 2).reshape(b, n, s.n_kv_heads, s.head_dim)
    kr = llama.rope(kn, pos, inv).reshape(b, n, -1).transpose(1, 0, 2)
    assert np.abs(qo - qr).max() < 4e-3 * np.abs(qr).max()
    assert np.abs(ko[past:] - kr).max() < 4e-3 * np.abs(kr).max()
    assert np.array_equal(ko[:past], k[:past].astype(np.float32))      # older positions untouched


@pytest.mark.parametrize("hd,H,Hkv,n,past", [(64, 8, 2, 1, 37), (128, 8, 4, 1, 300), (64, 8, 1, 1, 0),
                                             (64, 8, 2, 70, 0), (128, 4, 2, 33, 12), (128, 16, 2, 1, 100),
                                             (128, 32, 8, 1, 527), (64, 16, 4, 1, 5), (128, 64, 8, 1, 1039),
                                             (64, 32, 4, 1, 33), (128, 16, 8, 1, 16)])
@pytest.mark.parametrize("variant", [0, 5, 6])
def test_gqa_attention_vs_oracle(hd, H, Hkv, n, past, variant):
    """GQA attention (decode: the tensor-core kernel — variant 0 the production choice, 5 / 6
    forced to 4 / 2 warps — position splits + merge when the (b, KV head) pairs do not cover the
    SMs, ragged last tiles; prefill: the causal kernel)."""
    if n > 1 and variant:
        pytest.skip("variants select decode kernels")
    pipo = pipo_mod()
    rng = np.random.default_rng(hd + H + n + past)
    b = 3
    q = (rng.standard_normal((b, n, H * hd)) * hd ** -0.5).astype(np.float16)
    k = rng.standard_normal((past + n, b, Hkv * hd)).astype(np.float16)
    v = rng.standard_normal((past + n, b, Hkv * hd)).astype(np.float16)
    cfg = pipo.make_config(TINY, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE)
    with pipo.Pipeline(cfg) as pl:
        o = pipo.pipo_attention_gqa(pl.ctx, q, k, v, past, H, Hkv, variant)
    ref = llama.attention_gqa(q.astype(np.float64), k.astype(np.float64).transpose(1, 0, 2),
                              v.astype(np.float64).transpose(1, 0, 2), past, H, Hkv)
    assert rel_inf(o, ref) < 5e-3


def _teacher_forced(pipo, shape, emb, layers, wfmt, b, P, G, cfg_kw=None, capture=True):
    s_max = P + G
    ref = llama.OracleLlama.from_masters(shape, emb, layers, wfmt, s_max)
    cfg = pipo.make_config(shape, max_batch=b, max_seq=s_max,
                           wfmt=pipo.PIPO_W_INT4_G64 if wfmt == "int4" else pipo.PIPO_W_FP16,
                           **(cfg_kw or dict(weight_tier=pipo.PIPO_TIER_HOST)))
    prompt = synth.prompts(b, P, shape.vocab)
    errs = []
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        if capture:
            cap = np.zeros((shape.n_layers, b, P, shape.d_model), np.float32)
            pipo.pipo_debug_capture(pl.ctx, cap)
        _, lg = pl.prefill(prompt, want_logits=True)
        rl = ref.prefill(prompt)
        if capture:
            for j in range(shape.n_layers):
                assert rel_inf(cap[j], ref.capture[j]) < 2e-2, j
        errs.append(rel_inf(lg, rl))
        tok = np.argmax(rl, -1).astype(np.int32)
        for _ in range(G - 1):
            if capture:
                cap1 = np.zeros((shape.n_layers, b, 1, shape.d_model), np.float32)
                pipo.pipo_debug_capture(pl.ctx, cap1)
            nxt, lg = pl.decode_step(tok, want_logits=True)
            rl = ref.decode(tok)
            if capture:
                for j in range(shape.n_layers):
                    assert rel_inf(cap1[j], ref.capture[j]) < 2e-2, j
            errs.append(rel_inf(lg, rl))
            # ids equal wherever the oracle's top-2 margin is decided (reading Q11)
            srt = np.sort(rl, -1)
            decided = (srt[:, -1] - srt[:, -2]) >= 4 * np.abs(lg - rl).max()
            assert np.array_equal(nxt[decided], np.argmax(rl, -1)[decided])
            tok = np.argmax(rl, -1).astype(np.int32)
    assert max(errs) < 2e-2, errs
    return errs


@pytest.mark.parametrize("wfmt", ["int4", "fp16"])
@pytest.mark.parametrize("b", [3, 24])
def test_llama_tiny_vs_oracle(tiny, wfmt, b):
    pipo = pipo_mod()
    emb, layers = tiny
    _teacher_forced(pipo, TINY, emb, layers, wfmt, b, 20, 5)


def test_llama_hd128_vs_oracle():
    pipo = pipo_mod()
    emb, layers = _masters(TINY128)
    _teacher_forced(pipo, TINY128, emb, layers, "int4", 20, 24, 4)


def _logits_run(pipo, shape, loader, prompt, G, **cfg_kw):
    b, P = prompt.shape
    cfg = pipo.make_config(shape, max_batch=b, max_seq=P + G, **cfg_kw)
    out = []
    with pipo.Pipeline(cfg) as pl:
        loader(pl)
        nxt, lg = pl.prefill(prompt, want_logits=True)
        out.append(lg)
        for _ in range(G - 1):
            nxt, lg = pl.decode_step(nxt, want_logits=True)
            out.append(lg)
    return np.stack(out)


def test_llama_synthetic_loader_matches_masters(tiny):
    pipo = pipo_mod()
    emb, layers = tiny
    prompt = synth.prompts(20, 12, TINY.vocab)
    a = _logits_run(pipo, TINY, lambda pl: load_masters(pl, emb, layers), prompt, 3, weight_tier=pipo.PIPO_TIER_HOST)

    def syn(pl):
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, synth.WEIGHT_SEED)
        for j in range(TINY.n_layers):
            pl.load_synthetic(j, synth.WEIGHT_SEED)
    b = _logits_run(pipo, TINY, syn, prompt, 3, weight_tier=pipo.PIPO_TIER_HOST)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("variant", [dict(weight_tier=0), dict(weight_tier=1, ring_layers=1),
                                     dict(weight_tier=1, ring_layers=2, chunk_bytes=1 << 18),
                                     dict(weight_tier=1, kv_tier=1)])
def test_llama_tier_invariance(tiny, variant):
    pipo = pipo_mod()
    emb, layers = tiny
    prompt = synth.prompts(20, 10, TINY.vocab)
    load = lambda pl: load_masters(pl, emb, layers)
    base = _logits_run(pipo, TINY, load, prompt, 4, weight_tier=pipo.PIPO_TIER_HOST)
    other = _logits_run(pipo, TINY, load, prompt, 4, **variant)
    assert np.array_equal(base, other)


def test_llama_rejects_int4_kv():
    pipo = pipo_mod()
    cfg = pipo.make_config(TINY, max_batch=2, max_seq=8, kv_fmt=pipo.PIPO_W_INT4_G64)
    with pytest.raises(pipo.PipoError):
        pipo.Pipeline(cfg)


def test_llama_disk_tier_bit_identical(tiny, tmp_path):
    """LLaMA through the DISK tier (blob files -> reader pool -> pinned ring -> H2D):
    same logits as the HOST tier."""
    pipo = pipo_mod()
    prompt = synth.prompts(20, 10, TINY.vocab)

    def syn(pl):
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, synth.WEIGHT_SEED)
        for j in range(TINY.n_layers):
            pl.load_synthetic(j, synth.WEIGHT_SEED)
    base = _logits_run(pipo, TINY, syn, prompt, 4, weight_tier=pipo.PIPO_TIER_HOST)
    got = _logits_run(pipo, TINY, syn, prompt, 4, weight_tier=pipo.PIPO_TIER_DISK, disk_dir=str(tmp_path),
                      chunk_bytes=1 << 18, disk_threads=3)
    assert np.array_equal(base, got)


def test_llama_sharded_stream_world1_bit_identical(tiny):
    """NEXT-1 sharded streaming (1-rank NCCL all-gather) on the LLaMA path."""
    pipo = pipo_mod()
    emb, layers = tiny
    prompt = synth.prompts(20, 10, TINY.vocab)
    base = _logits_run(pipo, TINY, lambda pl: load_masters(pl, emb, layers), prompt, 4, weight_tier=pipo.PIPO_TIER_HOST)

    def sharded(pl):
        pipo.pipo_shard_stream_init(pl.ctx, 0, 1, pipo.pipo_nccl_unique_id())
        load_masters(pl, emb, layers)
    got = _logits_run(pipo, TINY, sharded, prompt, 4, weight_tier=pipo.PIPO_TIER_HOST)
    assert np.array_equal(base, got)
