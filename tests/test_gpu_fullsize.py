"""Full-size sampled parity: the kernels at the exact shapes and launch configurations
bench.py times (c5 OPT-30B: d = 7168, F = 28672, 56 heads, b = 64, P = 512, L up to 543;
c6 LLaMA3.1-8B: d = 4096, F = 14336, GQA 32/8), checked against the oracle's
definitions on SAMPLED outputs the fp64 oracle computes one by one (selected output
features / rows / sequences), since a full fp64 OPT-30B forward is out of reach.

The decode linears go through PATH_AUTO at M = 64 — the stream-K tcgen05 kernel the
pipeline launches — and the prefill linear through the persistent tcgen05 kernel at
M = b * P = 32768.  Output-feature groups are independent in the int4 encoding (one
scale per 64 weights of a row), so quantizing only the sampled rows on the oracle side
is exactly the full quantization restricted to those rows.
"""
import numpy as np
import pytest

from oracle import llama, opt, quant
from tests.gpu_util import check_greedy_ids, free_running, pipo_mod, rel_inf

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def env():
    pipo = pipo_mod()
    import pipo_synth as synth
    shape = synth.OPTShape(d_model=256, n_layers=1, n_heads=4, ffn_dim=512, vocab=512, max_pos=64)
    pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
    yield pipo, pl
    pl.close()


def _sampled_linear_check(pipo, pl, M, N, K, path, seed, n_rows=384, m_rows=None, tol=2e-3, wfmt=1):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((M, K), dtype=np.float32).astype(np.float16)
    w = (rng.standard_normal((N, K), dtype=np.float32) * np.float32(0.02)).astype(np.float16).astype(np.float32)
    bias = rng.uniform(-0.02, 0.02, N).astype(np.float32)
    y = pipo.pipo_linear(pl.ctx, wfmt, path, x, w, bias)
    rows = np.sort(rng.choice(N, n_rows, replace=False))
    rows[0], rows[-1] = 0, N - 1                              # first and last (ragged) tile
    ms = np.arange(M) if m_rows is None else np.sort(rng.choice(M, m_rows, replace=False))
    wsel = np.ascontiguousarray(w[rows])
    wh = (quant.quant_dequant(wsel) if wfmt == 1 else wsel).astype(np.float64)
    ref = x[ms].astype(np.float64) @ wh.T + bias[rows].astype(np.float16).astype(np.float64)
    err = rel_inf(y[np.ix_(ms, rows)], ref)
    assert err < 2e-2 and err < tol, (M, N, K, err)


@pytest.mark.parametrize("name,N,K", [("c5_qkv", 21504, 7168), ("c5_out", 7168, 7168), ("c5_fc1", 28672, 7168),
                                      ("c5_fc2", 7168, 28672), ("c6_qkv", 6144, 4096), ("c6_fc1", 28672, 4096),
                                      ("c6_fc2", 4096, 14336)])
def test_decode_linear_fullsize(env, name, N, K):
    pipo, pl = env
    _sampled_linear_check(pipo, pl, 64, N, K, pipo.PATH_AUTO, N + K)


@pytest.mark.parametrize("name,M,N,K", [("c5_head", 64, 50272, 7168), ("c6_head", 64, 128256, 4096),
                                        ("c7_head", 1, 128256, 4096)])
def test_lm_head_fullsize(env, name, M, N, K):
    """The LM head (a13) at the c5 / c6 / c7 shapes through the streaming fp16 tcgen05
    kernel the pipeline launches (PATH_HEAD), sampled vocabulary rows against fp64."""
    pipo, pl = env
    _sampled_linear_check(pipo, pl, M, N, K, pipo.PATH_HEAD, N + 1, wfmt=0, tol=1e-4)


def test_decode_linear_fullsize_b1_gemv(env):
    """c7 (b = 1): the CUDA-core GEMV at the LLaMA3.1-8B FC1 shape."""
    pipo, pl = env
    _sampled_linear_check(pipo, pl, 1, 28672, 4096, pipo.PATH_AUTO, 17)


def test_prefill_linear_fullsize_sampled(env):
    """c5 prefill out-proj: M = 64 x 512 tokens through the persistent tcgen05 kernel,
    checked on 96 sampled token rows x 384 sampled features."""
    pipo, pl = env
    _sampled_linear_check(pipo, pl, 64 * 512, 7168, 7168, pipo.PATH_AUTO, 5, n_rows=384, m_rows=96)


def test_decode_attention_fullsize(env):
    """c5 decode attention: b = 64, 56 heads x 128, L = 528 (mid-generation), 8 sampled
    sequences against the fp64 definition."""
    pipo, pl = env
    rng = np.random.default_rng(11)
    b, L, d, H = 64, 528, 7168, 56
    q = (rng.standard_normal((b, d), dtype=np.float32) * (d // H) ** -0.5).astype(np.float16)
    k = rng.standard_normal((L, b, d), dtype=np.float32).astype(np.float16)
    v = rng.standard_normal((L, b, d), dtype=np.float32).astype(np.float16)
    o = pipo.pipo_attention_decode(pl.ctx, q, k, v, H)
    seqs = np.array([0, 9, 17, 31, 32, 40, 55, 63])
    ref = opt.attention(q[seqs].astype(np.float64)[:, None], k[:, seqs].astype(np.float64).transpose(1, 0, 2),
                        v[:, seqs].astype(np.float64).transpose(1, 0, 2), L - 1, H)[:, 0]
    assert rel_inf(o[seqs], ref) < 5e-3


def test_gqa_decode_attention_fullsize(env):
    """c6 decode attention: b = 64, 32 query heads over 8 KV heads x 128, L = 528."""
    pipo, pl = env
    rng = np.random.default_rng(12)
    b, L, H, Hkv, hd = 64, 528, 32, 8, 128
    q = (rng.standard_normal((b, 1, H * hd), dtype=np.float32) * hd ** -0.5).astype(np.float16)
    k = rng.standard_normal((L, b, Hkv * hd), dtype=np.float32).astype(np.float16)
    v = rng.standard_normal((L, b, Hkv * hd), dtype=np.float32).astype(np.float16)
    o = pipo.pipo_attention_gqa(pl.ctx, q, k, v, L - 1, H, Hkv)
    seqs = np.array([0, 13, 38, 63])
    ref = llama.attention_gqa(q[seqs].astype(np.float64), k[:, seqs].astype(np.float64).transpose(1, 0, 2),
                              v[:, seqs].astype(np.float64).transpose(1, 0, 2), L - 1, H, Hkv)
    assert rel_inf(o[seqs], ref) < 5e-3


def test_prefill_attention_fullsize_sampled(env):
    """c5 prefill attention (causal, tensor-core kernel): b = 64, P = 512, 56 heads;
    2 sampled sequences against the fp64 definition."""
    pipo, pl = env
    rng = np.random.default_rng(13)
    b, n, d, H = 64, 512, 7168, 56
    q = (rng.standard_normal((b, n, d), dtype=np.float32) * (d // H) ** -0.5).astype(np.float16)
    k = rng.standard_normal((n, b, d), dtype=np.float32).astype(np.float16)
    v = rng.standard_normal((n, b, d), dtype=np.float32).astype(np.float16)
    o = pipo.pipo_attention_prefill(pl.ctx, q, k, v, 0, H)
    seqs = np.array([5, 62])
    ref = opt.attention(q[seqs].astype(np.float64), k[:, seqs].astype(np.float64).transpose(1, 0, 2),
                        v[:, seqs].astype(np.float64).transpose(1, 0, 2), 0, H)
    assert rel_inf(o[seqs], ref) < 1e-2


def test_c2_full_model_sampled_sequences():
    """configs[1] end to end: OPT-1.3B (24 layers, d = 2048), b = 16, P = 256, weights in
    pinned host memory (streamed), through prefill + 3 decode steps.  Sequences are
    independent, so the fp64 oracle runs only 2 sampled sequences of the batch; their
    per-layer outputs (debug capture) and logits must be within 2e-2 of the oracle.  The
    GPU is fed the oracle's greedy tokens for the sampled sequences (teacher forcing,
    reading Q11) and its own for the rest."""
    import pipo_synth as synth
    from tests.gpu_util import load_masters
    pipo = pipo_mod()
    s = synth.OPT_1_3B
    b, P, G = 16, 256, 4
    seqs = np.array([3, 12])
    emb = synth.embed_masters(s)
    layers = [synth.layer_masters(s, j) for j in range(s.n_layers)]
    ref = opt.OracleOPT.from_masters(s.n_heads, emb, layers, "int4", P + G)
    prompt = synth.prompts(b, P, s.vocab)
    cfg = pipo.make_config(s, max_batch=b, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST)
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        del layers
        cap = np.zeros((s.n_layers, b, P, s.d_model), np.float32)
        pipo.pipo_debug_capture(pl.ctx, cap)
        nxt, lg = pl.prefill(prompt, want_logits=True)
        rl = ref.prefill(prompt[seqs])
        for j in (0, s.n_layers // 2, s.n_layers - 1):
            assert rel_inf(cap[j][seqs], ref.capture[j]) < 2e-2, j
        assert rel_inf(lg[seqs], rl) < 2e-2
        und = check_greedy_ids(nxt[seqs], lg[seqs], rl, "prefill")
        for t in range(G - 1):
            tok = nxt.copy()
            tok[seqs] = np.argmax(rl, -1)
            nxt, lg = pl.decode_step(tok.astype(np.int32), want_logits=True)
            rl = ref.decode(tok[seqs])
            err = rel_inf(lg[seqs], rl)
            assert err < 2e-2, err
            und += check_greedy_ids(nxt[seqs], lg[seqs], rl, f"decode {t}")
        print("undecided", und, "of", G * len(seqs))


def test_c6_llama8b_two_layers_sampled_sequences():
    """c6 shapes end to end (LLaMA3.1-8B: d = 4096, GQA 32/8, SwiGLU 14336, V = 128256,
    llama3 RoPE), 2 of the 32 decoder layers (the per-layer kernels and launch
    configurations are the ones c6 runs), b = 64, P = 512, host-streamed int4 weights,
    prefill + 3 decode steps; 3 sampled sequences against the fp64 oracle, logits within
    2e-2 and the GPU argmax kernel's ids equal wherever decided (check_greedy_ids)."""
    import dataclasses

    import pipo_synth as synth
    from tests.gpu_util import load_masters
    pipo = pipo_mod()
    s = dataclasses.replace(synth.LLAMA31_8B, n_layers=2, max_pos=4096)
    b, P, G = 64, 512, 4
    seqs = np.array([7, 29, 50])
    emb = synth.llama_embed_masters(s)
    layers = [synth.llama_layer_masters(s, j) for j in range(s.n_layers)]
    ref = llama.OracleLlama.from_masters(s, emb, layers, "int4", P + G)
    prompt = synth.prompts(b, P, s.vocab)
    cfg = pipo.make_config(s, max_batch=b, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST)
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        del layers
        cap = np.zeros((s.n_layers, b, P, s.d_model), np.float32)
        pipo.pipo_debug_capture(pl.ctx, cap)
        nxt, lg = pl.prefill(prompt, want_logits=True)
        rl = ref.prefill(prompt[seqs])
        for j in range(s.n_layers):
            assert rel_inf(cap[j][seqs], ref.capture[j]) < 2e-2, j
        assert rel_inf(lg[seqs], rl) < 2e-2
        und = check_greedy_ids(nxt[seqs], lg[seqs], rl, "prefill")
        for t in range(G - 1):
            tok = nxt.copy()
            tok[seqs] = np.argmax(rl, -1)
            nxt, lg = pl.decode_step(tok.astype(np.int32), want_logits=True)
            rl = ref.decode(tok[seqs])
            assert rel_inf(lg[seqs], rl) < 2e-2
            und += check_greedy_ids(nxt[seqs], lg[seqs], rl, f"decode {t}")
        print("undecided", und, "of", G * len(seqs))


def test_c5_opt30b_two_layers_sampled_sequences():
    """The headline config's shapes end to end (OPT-30B: d = 7168, 56 heads, F = 28672,
    V = 50272), 2 of the 48 decoder layers, b = 64, P = 512, host-streamed int4 weights,
    prefill + 3 decode steps; 3 sampled sequences against the fp64 oracle, logits within
    2e-2 and the GPU argmax kernel's ids equal wherever decided (check_greedy_ids)."""
    import dataclasses

    import pipo_synth as synth
    from tests.gpu_util import load_masters
    pipo = pipo_mod()
    s = dataclasses.replace(synth.OPT_30B, n_layers=2)
    b, P, G = 64, 512, 4
    seqs = np.array([1, 33, 60])
    emb = synth.embed_masters(s)
    layers = [synth.layer_masters(s, j) for j in range(s.n_layers)]
    ref = opt.OracleOPT.from_masters(s.n_heads, emb, layers, "int4", P + G)
    prompt = synth.prompts(b, P, s.vocab)
    cfg = pipo.make_config(s, max_batch=b, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST)
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        del layers
        cap = np.zeros((s.n_layers, b, P, s.d_model), np.float32)
        pipo.pipo_debug_capture(pl.ctx, cap)
        nxt, lg = pl.prefill(prompt, want_logits=True)
        rl = ref.prefill(prompt[seqs])
        for j in range(s.n_layers):
            assert rel_inf(cap[j][seqs], ref.capture[j]) < 2e-2, j
        assert rel_inf(lg[seqs], rl) < 2e-2
        und = check_greedy_ids(nxt[seqs], lg[seqs], rl, "prefill")
        for t in range(G - 1):
            tok = nxt.copy()
            tok[seqs] = np.argmax(rl, -1)
            nxt, lg = pl.decode_step(tok.astype(np.int32), want_logits=True)
            rl = ref.decode(tok[seqs])
            assert rel_inf(lg[seqs], rl) < 2e-2
            und += check_greedy_ids(nxt[seqs], lg[seqs], rl, f"decode {t}")
        print("undecided", und, "of", G * len(seqs))


@pytest.mark.parametrize("tier", ["device", "host"])
def test_synthetic_loader_bytes_at_c5_shapes(tier):
    """The bench's weights (pipo_load_synthetic: the library's GPU generator + GPU
    quantizer, then the tier's store) at the c5 tensor sizes — FC1 and FC2 hold
    205 M weights, the token table 360 M values — equal, byte for byte on sampled
    rows, the numpy masters (pipo_synth) quantized by the oracle (oracle/quant.py):
    int4 codes, fp16 scale bits, and the fp16 embedding rows."""
    import dataclasses

    import pipo_synth as synth
    pipo = pipo_mod()
    s = dataclasses.replace(synth.OPT_30B, n_layers=1)
    d, F = s.d_model, s.ffn_dim
    cfg = pipo.make_config(s, max_batch=1, max_seq=2, weight_tier=0 if tier == "device" else 1)
    rng = np.random.default_rng(5)
    with pipo.Pipeline(cfg) as pl:
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, synth.WEIGHT_SEED)
        pl.load_synthetic(0, synth.WEIGHT_SEED)
        for m, (tid, N, K) in enumerate([(synth.T_W_QKV, 3 * d, d), (synth.T_W_OUT, d, d),
                                         (synth.T_W_FC1, F, d), (synth.T_W_FC2, d, F)]):
            rows = np.unique(np.concatenate([[0, N - 1], rng.choice(N, 6, replace=False)]))
            w = synth.draw_rows(synth.WEIGHT_SEED, 1, tid, synth.KIND_NORMAL, synth.W_STD, K, rows)
            q, sc = quant.quantize_int4_g64(w)
            for i, r in enumerate(rows):
                codes, scales = pipo.pipo_debug_read_rows(pl.ctx, 0, m, int(r), 1, K, True)
                assert np.array_equal(codes[0], quant.pack_int4(q[i:i + 1])[0]), (m, r)
                assert np.array_equal(scales[0], quant.scales_to_bits(sc[i:i + 1])[0]), (m, r)
        rows = np.unique(np.concatenate([[0, s.vocab - 1], rng.choice(s.vocab, 6, replace=False)]))
        want = synth.draw_rows(synth.WEIGHT_SEED, 0, synth.T_TOK, synth.KIND_NORMAL, synth.W_STD, d, rows)
        for i, r in enumerate(rows):
            got = pipo.pipo_debug_read_rows(pl.ctx, pipo.PIPO_LAYER_EMBED, 0, int(r), 1, d, False)
            assert np.array_equal(got[0].view(np.uint16), want[i].astype(np.float16).view(np.uint16)), r


def test_c2_free_running_greedy_ids():
    """configs[1] (OPT-1.3B, 24 layers, b = 16, P = 256) generated FREE-RUNNING for all
    G = 32 tokens: the GPU feeds back its own ids (whole batch), the fp64 oracle its own
    for two sequences.  The sequences come from tests/golden/c2_free_running.json
    (written by a committed script that calls only oracle/): sequence 10 is the one whose
    32 oracle steps all have top-2 margins > 0.026 (logits up to 4.5), so every step is
    decided and all 32 ids must be equal (reading Q11's fixture rule); sequence 1 (min
    margin 0.0089) must agree at every decided step and may only diverge at a near tie.
    The golden ids themselves are re-derived live by the oracle (no stored value is
    trusted for the comparison)."""
    import json
    import os

    import pipo_synth as synth
    from tests.gpu_util import load_masters
    pipo = pipo_mod()
    s = synth.OPT_1_3B
    b, P, G = 16, 256, 32
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c2_free_running.json")))
    exact, other = 10, 1
    assert min(gold["margins"][exact]) > 0.02
    emb = synth.embed_masters(s)
    layers = [synth.layer_masters(s, j) for j in range(s.n_layers)]
    ref = opt.OracleOPT.from_masters(s.n_heads, emb, layers, "int4", P + G)
    prompt = synth.prompts(b, P, s.vocab)
    cfg = pipo.make_config(s, max_batch=b, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST)
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        del layers
        ids_g, ids_r, n_und, n_div = free_running(pl, ref, prompt, G, rows=[exact, other])
    print(f"undecided {n_und}, diverged {n_div}")
    assert np.array_equal(ids_r[0], gold["ids"][exact])           # the live oracle reproduces the fixture
    assert np.array_equal(ids_g[exact], ids_r[0])                  # 32 free-running ids, exactly
    agree = (ids_g == np.asarray(gold["ids"])).all(axis=1)
    print("sequences whose 32 GPU ids equal the oracle's:", int(agree.sum()), "of", b)
