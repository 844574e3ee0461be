"""Pins for oracle/opt.py against things other than itself.

* transformers' OPTForCausalLM (float64, tiny config) loaded with the SAME
  dequantized weights: the library's independent implementation of the OPT block
  ([ext] modeling_opt.py) — logits agree to ~1e-12 and greedy ids are identical,
  for prefill and for cached decode.
* brute-force attention with explicit Python loops over (b, head, t, position).
* special cases: one cached position -> output = that V row;
  all-equal keys -> mean of V; softmax rows sum to 1.
* LayerNorm of a constant row is beta exactly; vs statistics-module closed form.
* KV-cache consistency: prefill(P) + decode(t) == prefill(P + 1) at the last position.
* causality: logits at t do not depend on tokens after t.
"""
import math
import statistics

import numpy as np
import pytest

import pipo_synth as synth
from oracle import opt, quant

TINY = synth.OPTShape(d_model=64, n_layers=2, n_heads=4, ffn_dim=256, vocab=512, max_pos=64)


def _tiny_model(wfmt="int4", s_max=48, seed=synth.WEIGHT_SEED):
    emb = synth.embed_masters(TINY, seed)
    layers = [synth.layer_masters(TINY, j, seed) for j in range(TINY.n_layers)]
    return opt.OracleOPT.from_masters(TINY.n_heads, emb, layers, wfmt, s_max), emb, layers


def _hf_model(model: opt.OracleOPT):
    torch = pytest.importorskip("torch")
    transformers = pytest.importorskip("transformers")
    cfg = transformers.OPTConfig(
        vocab_size=TINY.vocab, hidden_size=TINY.d_model, num_hidden_layers=TINY.n_layers,
        ffn_dim=TINY.ffn_dim, num_attention_heads=TINY.n_heads, max_position_embeddings=TINY.max_pos,
        do_layer_norm_before=True, word_embed_proj_dim=TINY.d_model, dropout=0.0,
        attention_dropout=0.0, activation_function="relu", enable_bias=True,
        layer_norm_elementwise_affine=True, tie_word_embeddings=True, pad_token_id=1)
    cfg._attn_implementation = "sdpa"   # eager casts softmax to fp32; sdpa stays fp64
    m = transformers.OPTForCausalLM(cfg).to(torch.float64).eval()
    d = TINY.d_model
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    with torch.no_grad():
        dec = m.model.decoder
        dec.embed_tokens.weight.copy_(t(model.tok))
        dec.embed_positions.weight.copy_(t(model.pos))
        dec.final_layer_norm.weight.copy_(t(model.lnf_g))
        dec.final_layer_norm.bias.copy_(t(model.lnf_b))
        for lay, w in zip(dec.layers, model.layers):
            sa = lay.self_attn
            for name, sl in (("q_proj", slice(0, d)), ("k_proj", slice(d, 2 * d)), ("v_proj", slice(2 * d, 3 * d))):
                getattr(sa, name).weight.copy_(t(w.w_qkv[sl]))
                getattr(sa, name).bias.copy_(t(w.b_qkv[sl]))
            sa.out_proj.weight.copy_(t(w.w_out)); sa.out_proj.bias.copy_(t(w.b_out))
            lay.self_attn_layer_norm.weight.copy_(t(w.ln1_g)); lay.self_attn_layer_norm.bias.copy_(t(w.ln1_b))
            lay.final_layer_norm.weight.copy_(t(w.ln2_g)); lay.final_layer_norm.bias.copy_(t(w.ln2_b))
            lay.fc1.weight.copy_(t(w.w_fc1)); lay.fc1.bias.copy_(t(w.b_fc1))
            lay.fc2.weight.copy_(t(w.w_fc2)); lay.fc2.bias.copy_(t(w.b_fc2))
        assert m.lm_head.weight.data_ptr() == dec.embed_tokens.weight.data_ptr() or \
            torch.equal(m.lm_head.weight, dec.embed_tokens.weight)
    return m, torch


@pytest.mark.parametrize("wfmt", ["int4", "fp16"])
def test_oracle_matches_hf_opt(wfmt):
    model, _, _ = _tiny_model(wfmt)
    hf, torch = _hf_model(model)
    ids = synth.prompts(2, 12, TINY.vocab)
    ref_all = model.forward(ids, all_logits=True)           # [2, 12, V]
    with torch.no_grad():
        out = hf(input_ids=torch.from_numpy(ids.astype(np.int64)), use_cache=True)
    hf_all = out.logits.numpy()
    rel = np.abs(ref_all - hf_all).max() / np.abs(hf_all).max()
    assert rel < 1e-10, rel
    # cached decode, 4 greedy steps, both sides on their own caches
    past = out.past_key_values
    nxt = opt.greedy(ref_all[:, -1])
    assert np.array_equal(nxt, hf_all[:, -1].argmax(-1))
    for _ in range(4):
        ref = model.decode(nxt)
        with torch.no_grad():
            o = hf(input_ids=torch.from_numpy(nxt.astype(np.int64)[:, None]), past_key_values=past, use_cache=True)
        past = o.past_key_values
        h = o.logits[:, -1].numpy()
        assert np.abs(ref - h).max() / np.abs(h).max() < 1e-10
        assert np.array_equal(opt.greedy(ref), h.argmax(-1))
        nxt = opt.greedy(ref)


def test_int4_weights_are_quant_dequant():
    model, _, layers = _tiny_model("int4")
    w = layers[1]["w_fc2"]
    assert np.array_equal(model.layers[1].w_fc2, quant.quant_dequant(w).astype(np.float64))
    assert np.array_equal(model.layers[1].b_fc2, layers[1]["b_fc2"].astype(np.float64))


def _brute_attention(q, k, v, past, H):
    b, n, d = q.shape
    hd = d // H
    o = np.zeros_like(q)
    for bi in range(b):
        for h in range(H):
            sl = slice(h * hd, (h + 1) * hd)
            for t in range(n):
                L = past + t + 1
                sc = [sum(q[bi, t, sl][i] * k[bi, p, sl][i] for i in range(hd)) for p in range(L)]
                m = max(sc)
                e = [math.exp(x - m) for x in sc]
                z = sum(e)
                for i in range(hd):
                    o[bi, t, h * hd + i] = sum(e[p] / z * v[bi, p, h * hd + i] for p in range(L))
    return o


@pytest.mark.parametrize("past,n", [(0, 5), (4, 1), (3, 3)])
def test_attention_brute_force(past, n):
    rng = np.random.default_rng(past * 10 + n)
    b, H, hd = 2, 2, 4
    q = rng.standard_normal((b, n, H * hd))
    k = rng.standard_normal((b, past + n + 2, H * hd))
    v = rng.standard_normal((b, past + n + 2, H * hd))
    got = opt.attention(q, k, v, past, H)
    ref = _brute_attention(q, k, v, past, H)
    assert np.abs(got - ref).max() < 1e-12


def test_attention_special_cases():
    rng = np.random.default_rng(7)
    q = rng.standard_normal((1, 1, 8))
    k = rng.standard_normal((1, 6, 8))
    v = rng.standard_normal((1, 6, 8))
    # one cached position: softmax over one logit is 1 -> output is that V row
    assert np.array_equal(opt.attention(q, k, v, 0, 2)[0, 0], v[0, 0])
    # all-equal keys -> uniform weights -> mean of V rows
    k2 = np.repeat(k[:, :1], 6, axis=1)
    got = opt.attention(q, k2, v, 5, 2)[0, 0]
    assert np.abs(got - v[0].mean(axis=0)).max() < 1e-14
    s = opt.softmax(rng.standard_normal((5, 9)) * 10)
    assert np.abs(s.sum(-1) - 1).max() < 1e-12


def test_layer_norm_closed_form():
    g = np.linspace(0.5, 1.5, 16)
    b = np.linspace(-1, 1, 16)
    assert np.array_equal(opt.layer_norm(np.full((1, 16), 3.25), g, b)[0], b)
    x = np.random.default_rng(3).standard_normal(16)
    mu = statistics.fmean(x)
    var = statistics.pvariance(x)
    ref = [(xi - mu) / math.sqrt(var + 1e-5) * gi + bi for xi, gi, bi in zip(x, g, b)]
    assert np.abs(opt.layer_norm(x[None], g, b)[0] - ref).max() < 1e-12


def test_kv_cache_consistency():
    m1, _, _ = _tiny_model()
    m2, _, _ = _tiny_model()
    ids = synth.prompts(3, 9, TINY.vocab)
    m1.prefill(ids[:, :8])
    a = m1.decode(ids[:, 8])
    b = m2.prefill(ids)
    assert np.abs(a - b).max() / np.abs(b).max() < 1e-12


def test_causality():
    m, _, _ = _tiny_model()
    ids = synth.prompts(1, 10, TINY.vocab)
    a = m.forward(ids, all_logits=True)
    ids2 = ids.copy()
    ids2[0, 6:] = (ids2[0, 6:] + 17) % TINY.vocab
    m.past = 0
    b = m.forward(ids2, all_logits=True)
    assert np.array_equal(a[0, :6], b[0, :6])
    assert not np.array_equal(a[0, 6:], b[0, 6:])


def test_generate_prefill_then_decode_steps():
    m, _, _ = _tiny_model()
    ids, logits = opt.generate(m, synth.prompts(2, 6, TINY.vocab), 5)
    assert ids.shape == (2, 5) and len(logits) == 5
    assert m.past == 6 + 4       # prefill 6 positions, then G-1 = 4 decode steps


def test_int4_kv_cache_semantics():
    """INT4 KV (reading Q17b): prefill logits are untouched (fresh K/V), the cache
    holds exactly the weight encoder's quant->dequant of the fresh rows, and a decode
    step reads that cache; its logits stay within the 4-bit error of the fp KV path."""
    m_fp, _, _ = _tiny_model()
    m_q = opt.OracleOPT.from_masters(TINY.n_heads, synth.embed_masters(TINY),
                                     [synth.layer_masters(TINY, j) for j in range(TINY.n_layers)],
                                     "int4", 48, kv_int4=True)
    ids = synth.prompts(2, 10, TINY.vocab)
    a = m_fp.prefill(ids)
    b = m_q.prefill(ids)
    assert np.array_equal(a, b)
    for j in range(TINY.n_layers):
        # the fp path's cache row and the int4 path's cache row come from the same fresh K
        assert np.array_equal(m_q.kc[j][:, :10], opt.kv_quant_dequant(m_fp.kc[j][:, :10]))
    nxt = opt.greedy(a)
    da = m_fp.decode(nxt)
    db = m_q.decode(nxt)
    rel = np.abs(da - db).max() / np.abs(da).max()
    assert 0 < rel < 0.2
    # one cached position per sequence: attention output = the dequantized V row
    q = np.random.default_rng(1).standard_normal((1, 1, 64))
    v = opt.kv_quant_dequant(np.random.default_rng(2).standard_normal((1, 1, 64)))
    assert np.array_equal(opt.attention(q, v, v, 0, 1)[0, 0], v[0, 0])


def test_int4_kv_decode_reads_own_row_quantized():
    """Reading Q17b pinned on a hand-built model (tests/q17b_model.py) where the two
    readings differ by 0.063 per element: the decode step's output equals the closed
    form in which its OWN new V row is read back quantize->dequantized (reading A),
    and is far from the form that keeps the own row in full precision (reading B)."""
    from tests import q17b_model as qm
    emb, layers = qm.masters()
    m = opt.OracleOPT.from_masters(1, emb, layers, "int4", 4, kv_int4=True)
    m.prefill(qm.prompt())
    m.decode(qm.decode_tokens())
    got = m.capture[0][:, 0]                                      # [b, d] layer output
    c = float(quant.quant_dequant(np.eye(64, dtype=np.float32))[0, 0])   # int4 identity = c I
    assert abs(c - 7 * 0.142822265625) < 1e-12                    # fp16_rne(1/7) * 7

    def ln(x):
        mu = x.mean()
        return (x - mu) / np.sqrt(((x - mu) ** 2).mean() + 1e-5)
    h0 = emb["tok"][qm.PROMPT_TOKEN].astype(np.float64)
    h1 = emb["tok"][qm.SPIKE_TOKEN].astype(np.float64)
    v0, v1 = c * ln(h0), c * ln(h1)
    dq = lambda v: quant.quant_dequant(v[None].astype(np.float32))[0].astype(np.float64)  # noqa: E731
    want_a = h1 + c * (dq(v0) + dq(v1)) / 2
    want_b = h1 + c * (dq(v0) + v1) / 2
    assert np.abs(got - want_a).max() < 1e-9
    assert np.abs(want_a - want_b)[1:].min() > 0.05               # the readings are far apart
    assert np.all(dq(v1)[1:] == 0)                                # the spike's small entries quantize to 0
