"""Pins for oracle/llama.py (NEXT-4) against things other than itself.

* transformers' LlamaForCausalLM (float64, tiny GQA config, llama3 rope scaling) with
  the SAME dequantized weights — the library's independent implementation of the
  LLaMA block: logits agree to ~1e-7 (HF's rotary embedding runs in fp32) and greedy
  ids are identical, prefill and cached decode.
* transformers' `_compute_llama3_parameters` (library routine) for the inverse
  frequencies, with the plain-RoPE special case theta^(-2i/hd) (factor = 0).
* RoPE invariants: position 0 is the identity; each (i, i + hd/2) pair keeps its
  norm; the score q(p)·k(p') depends only on p - p' (shifting both positions by the
  same amount leaves it unchanged) — a rotation property a sign or index slip breaks.
* brute-force GQA attention in explicit Python loops (query head j reads KV head
  j // group); h_kv = h reduces GQA to plain multi-head attention.
* RMSNorm: constant row c -> g * c / sqrt(c^2 + eps); vs the statistics module.
* SwiGLU pieces: silu(0) = 0, silu(x) -> x for large x, silu(-x) -> 0.
* KV-cache consistency: prefill(P) + decode == prefill(P + 1) at the last position.
"""
import math
import statistics

import numpy as np
import pytest

import pipo_synth as synth
from oracle import llama

TINY = synth.LlamaShape(d_model=64, n_layers=2, n_heads=4, n_kv_heads=2, ffn_dim=128, vocab=512, max_pos=64,
                        rope_theta=500000.0, rope_factor=8.0, rope_orig_max_pos=32)


def _tiny(wfmt="int4", s_max=48, shape=TINY):
    emb = synth.llama_embed_masters(shape)
    layers = [synth.llama_layer_masters(shape, j) for j in range(shape.n_layers)]
    return llama.OracleLlama.from_masters(shape, emb, layers, wfmt, s_max)


def _hf(model: llama.OracleLlama, shape=TINY):
    torch = pytest.importorskip("torch")
    transformers = pytest.importorskip("transformers")
    rope = {"rope_type": "llama3", "rope_theta": shape.rope_theta, "factor": shape.rope_factor,
            "low_freq_factor": shape.rope_low_freq, "high_freq_factor": shape.rope_high_freq,
            "original_max_position_embeddings": shape.rope_orig_max_pos}
    cfg = transformers.LlamaConfig(
        vocab_size=shape.vocab, hidden_size=shape.d_model, intermediate_size=shape.ffn_dim,
        num_hidden_layers=shape.n_layers, num_attention_heads=shape.n_heads,
        num_key_value_heads=shape.n_kv_heads, max_position_embeddings=shape.max_pos, rms_norm_eps=1e-5,
        rope_parameters=rope, attention_bias=False, mlp_bias=False, tie_word_embeddings=False,
        hidden_act="silu")
    cfg._attn_implementation = "sdpa"
    m = transformers.LlamaForCausalLM(cfg).to(torch.float64).eval()
    d, dkv, F = shape.d_model, shape.d_kv, shape.ffn_dim
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    with torch.no_grad():
        m.model.embed_tokens.weight.copy_(t(model.tok))
        m.model.norm.weight.copy_(t(model.lnf_g))
        m.lm_head.weight.copy_(t(model.lm_head))
        for lay, w in zip(m.model.layers, model.layers):
            sa = lay.self_attn
            sa.q_proj.weight.copy_(t(w.w_qkv[:d]))
            sa.k_proj.weight.copy_(t(w.w_qkv[d:d + dkv]))
            sa.v_proj.weight.copy_(t(w.w_qkv[d + dkv:]))
            sa.o_proj.weight.copy_(t(w.w_out))
            lay.input_layernorm.weight.copy_(t(w.ln1_g))
            lay.post_attention_layernorm.weight.copy_(t(w.ln2_g))
            lay.mlp.gate_proj.weight.copy_(t(w.w_fc1[:F]))
            lay.mlp.up_proj.weight.copy_(t(w.w_fc1[F:]))
            lay.mlp.down_proj.weight.copy_(t(w.w_fc2))
    return m


@pytest.mark.parametrize("wfmt", ["int4", "fp16"])
def test_matches_hf_llama_prefill_and_decode(wfmt):
    torch = pytest.importorskip("torch")
    model = _tiny(wfmt)
    hf = _hf(model)
    prompt = synth.prompts(2, 12, TINY.vocab)
    ours = [model.prefill(prompt)]
    ids = prompt.copy()
    for _ in range(4):
        nxt = np.argmax(ours[-1], axis=-1)
        ids = np.concatenate([ids, nxt[:, None]], axis=1)
        ours.append(model.decode(nxt))
    with torch.no_grad():
        ref = hf(torch.from_numpy(ids.astype(np.int64))).logits.numpy()
    for i, lg in enumerate(ours):
        r = ref[:, 11 + i]
        # HF computes inv_freq, p * inv_freq and cos/sin in fp32 (LlamaRotaryEmbedding);
        # angle error <= p * 2^-24 rad ~ 1e-6 here, far below any dropped term or sign slip
        assert np.abs(lg - r).max() <= 1e-6 * np.abs(r).max(), i
        assert np.array_equal(np.argmax(lg, -1), np.argmax(r, -1))


def test_inv_freq_matches_transformers_llama3_rule():
    torch = pytest.importorskip("torch")
    transformers = pytest.importorskip("transformers")
    from transformers.modeling_rope_utils import ROPE_INIT_FUNCTIONS
    for hd, theta, orig in ((128, 500000.0, 8192), (64, 10000.0, 32)):
        cfg = transformers.LlamaConfig(hidden_size=hd * 4, num_attention_heads=4, rope_parameters={
            "rope_type": "llama3", "rope_theta": theta, "factor": 8.0, "low_freq_factor": 1.0,
            "high_freq_factor": 4.0, "original_max_position_embeddings": orig})
        ref, _ = ROPE_INIT_FUNCTIONS["llama3"](cfg, torch.device("cpu"))
        ours = llama.rope_inv_freq(hd, theta, 8.0, 1.0, 4.0, orig)
        assert np.allclose(ours, ref.double().numpy(), rtol=1e-6, atol=0)   # HF computes in fp32
    plain = llama.rope_inv_freq(8, 10000.0)
    assert np.allclose(plain, [1.0, 10000.0 ** -0.25, 10000.0 ** -0.5, 10000.0 ** -0.75], rtol=1e-15)


def test_rope_invariants():
    rng = np.random.default_rng(0)
    inv = llama.rope_inv_freq(16, 500000.0, 8.0, 1.0, 4.0, 32)
    x = rng.standard_normal((1, 1, 1, 16))
    assert np.array_equal(llama.rope(x, np.array([0]), inv), x)
    y = llama.rope(x, np.array([37]), inv)
    assert np.allclose(x[..., :8] ** 2 + x[..., 8:] ** 2, y[..., :8] ** 2 + y[..., 8:] ** 2, rtol=1e-13)
    q, k = rng.standard_normal((2, 1, 1, 1, 16))
    for p, pk, shift in ((5, 2, 11), (30, 0, 100), (7, 7, 3)):
        s0 = (llama.rope(q, np.array([p]), inv) * llama.rope(k, np.array([pk]), inv)).sum()
        s1 = (llama.rope(q, np.array([p + shift]), inv) * llama.rope(k, np.array([pk + shift]), inv)).sum()
        assert abs(s0 - s1) <= 1e-12 * max(1.0, abs(s0))
    # hand-evaluated: hd = 2, inv = 1 -> a plain 2-D rotation by p radians
    z = llama.rope(np.array([[[[1.0, 0.0]]]]), np.array([1]), np.array([1.0]))
    assert np.allclose(z.ravel(), [math.cos(1.0), math.sin(1.0)], rtol=0, atol=1e-15)


def test_gqa_attention_brute_force():
    rng = np.random.default_rng(1)
    b, n, past, H, Hkv, hd = 2, 3, 4, 4, 2, 8
    q = rng.standard_normal((b, n, H * hd))
    k = rng.standard_normal((b, past + n, Hkv * hd))
    v = rng.standard_normal((b, past + n, Hkv * hd))
    got = llama.attention_gqa(q, k, v, past, H, Hkv)
    group = H // Hkv
    for bi in range(b):
        for j in range(H):
            g = j // group
            for t in range(n):
                L = past + t + 1
                s = [sum(q[bi, t, j * hd + e] * k[bi, p, g * hd + e] for e in range(hd)) for p in range(L)]
                mx = max(s)
                w = [math.exp(x - mx) for x in s]
                z = sum(w)
                for e in range(hd):
                    ref = sum(w[p] * v[bi, p, g * hd + e] for p in range(L)) / z
                    assert abs(got[bi, t, j * hd + e] - ref) < 1e-12
    # h_kv = h: each head reads its own K/V
    k2 = rng.standard_normal((b, past + n, H * hd))
    v2 = rng.standard_normal((b, past + n, H * hd))
    mha = llama.attention_gqa(q, k2, v2, past, H, H)
    one = llama.attention_gqa(q[..., :hd], k2[..., :hd], v2[..., :hd], past, 1, 1)
    assert np.allclose(mha[..., :hd], one, rtol=0, atol=1e-14)


def test_rmsnorm_and_silu():
    g = np.array([1.5, -0.5, 2.0, 1.0])
    c = 0.3
    out = llama.rms_norm(np.full(4, c), g)
    assert np.allclose(out, g * c / math.sqrt(c * c + 1e-5), rtol=1e-15)
    x = np.array([0.2, -1.0, 3.0, 0.7])
    ref = x / math.sqrt(statistics.fmean(float(v) ** 2 for v in x) + 1e-5)
    assert np.allclose(llama.rms_norm(x, np.ones(4)), ref, rtol=1e-14)
    assert llama.silu(np.array(0.0)) == 0.0
    assert abs(llama.silu(np.array(40.0)) - 40.0) < 1e-15
    assert abs(llama.silu(np.array(-40.0))) < 1e-15


def test_kv_cache_consistency():
    m1, m2 = _tiny(), _tiny()
    prompt = synth.prompts(2, 9, TINY.vocab)
    m1.prefill(prompt[:, :8])
    a = m1.decode(prompt[:, 8])
    b = m2.prefill(prompt)
    assert np.allclose(a, b, rtol=0, atol=1e-12 * np.abs(b).max())
