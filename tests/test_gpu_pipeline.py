"""GPU parity of the whole streamed-weight pipeline (prefill + decode) vs the oracle.

* c1 (BASELINE.json configs[0]): one OPT-125M-shaped decoder layer, int4 g64,
  b=4, P=32, gen 8 — every layer output (debug capture) and every step's logits
  within 2e-2 of the fp64 oracle, greedy ids equal wherever decided (Q11).
* the library's GPU generator + GPU quantizer (pipo_load_synthetic) reproduce the
  numpy masters + host quantizer bit-for-bit (identical logits);
* the method's invariance (the offloading changes nothing):
  DEVICE vs HOST tier, ring depths 1/2/3, chunk sizes -> bit-identical logits;
* host-resident KV (c3 mode) == device KV, bit-identical;
* GEMM path (b >= 16), hd = 64 and 128, fp16 weights, several layers.
"""
import numpy as np
import pytest

import pipo_synth as synth
from oracle import opt
from tests.gpu_util import assert_near_ties, free_running, load_masters, pipo_mod, rel_inf, teacher_forced

pytestmark = pytest.mark.gpu

C1 = synth.OPTShape(d_model=768, n_layers=1, n_heads=12, ffn_dim=3072)      # configs[0]


def _oracle(shape, emb, layers, wfmt, s_max):
    return opt.OracleOPT.from_masters(shape.n_heads, emb, layers, wfmt, s_max)


@pytest.fixture(scope="module")
def c1_masters():
    emb = synth.embed_masters(C1)
    layers = [synth.layer_masters(C1, 0)]
    return emb, layers


def test_c1_vs_oracle_layer_outputs_and_logits(c1_masters):
    pipo = pipo_mod()
    emb, layers = c1_masters
    b, P, G = 4, 32, 8
    prompt = synth.prompts(b, P, C1.vocab)
    ref = _oracle(C1, emb, layers, "int4", P + G)
    cfg = pipo.make_config(C1, max_batch=b, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST)
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        cap = np.zeros((1, b, P, C1.d_model), np.float32)
        pipo.pipo_debug_capture(pl.ctx, cap)
        _, lg = pl.prefill(prompt, want_logits=True)
        rl = ref.prefill(prompt)
        assert rel_inf(cap[0], ref.capture[0]) < 2e-2
        assert rel_inf(lg, rl) < 2e-2
        tok = opt.greedy(rl)
        for _ in range(G - 1):
            cap1 = np.zeros((1, b, 1, C1.d_model), np.float32)
            pipo.pipo_debug_capture(pl.ctx, cap1)
            _, lg = pl.decode_step(tok, want_logits=True)
            rl = ref.decode(tok)
            assert rel_inf(cap1[0], ref.capture[0]) < 2e-2
            assert rel_inf(lg, rl) < 2e-2
            tok = opt.greedy(rl)


# Reading Q11: "the committed fixture seed is also chosen so that free-running greedy
# ids match exactly".  At the default prompt seed (3664) two c1 oracle steps have
# top-2 margins of 1.7e-3 and 2.2e-3 (logits up to 3.0), i.e. ties within fp16
# arithmetic; 3667 is the first seed >= 3664 whose 32 oracle steps all have margins
# > 0.02 (min 0.040), so every step is decided and exact equality is a theorem.
C1_FREE_SEED = 3667


@pytest.mark.parametrize("seed", [C1_FREE_SEED, synth.PROMPT_SEED])
def test_c1_free_running_greedy_ids(c1_masters, seed):
    """Free-running greedy generation (each side feeds back its own ids).  At the
    fixture seed every step must be decided and all 4 x 8 ids equal; at the default
    seed decided steps must agree and a sequence may only diverge at a near tie."""
    pipo = pipo_mod()
    emb, layers = c1_masters
    b, P, G = 4, 32, 8
    prompt = synth.prompts(b, P, C1.vocab, seed=seed)
    cfg = pipo.make_config(C1, max_batch=b, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST)
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        ids_g, ids_r, n_und, n_div = free_running(pl, _oracle(C1, emb, layers, "int4", P + G), prompt, G)
    print(f"seed {seed}: undecided {n_und}, diverged {n_div}")
    if seed == C1_FREE_SEED:
        assert n_und == 0 and n_div == 0
        assert np.array_equal(ids_g, ids_r)


def _run(pipo, shape, cfg_kw, loader, prompt, G, want_logits=True, hook=None):
    b, P = prompt.shape
    cfg = pipo.make_config(shape, max_batch=b, max_seq=P + G, **cfg_kw)
    out = []
    with pipo.Pipeline(cfg) as pl:
        loader(pl)
        if hook is not None:
            hook(pl)
        nxt, lg = pl.prefill(prompt, want_logits=want_logits)
        out.append(lg)
        for _ in range(G - 1):
            nxt, lg = pl.decode_step(nxt, want_logits=want_logits)
            out.append(lg)
        st = pl.stats()
    return np.stack(out), st


def test_synthetic_loader_matches_masters(c1_masters):
    pipo = pipo_mod()
    emb, layers = c1_masters
    prompt = synth.prompts(4, 16, C1.vocab)
    a, _ = _run(pipo, C1, dict(weight_tier=pipo.PIPO_TIER_HOST), lambda pl: load_masters(pl, emb, layers), prompt, 3)
    def syn(pl):
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, synth.WEIGHT_SEED)
        pl.load_synthetic(0, synth.WEIGHT_SEED)
    b, _ = _run(pipo, C1, dict(weight_tier=pipo.PIPO_TIER_HOST), syn, prompt, 3)
    assert np.array_equal(a, b)


SMALL = synth.OPTShape(d_model=512, n_layers=4, n_heads=4, ffn_dim=2048, vocab=1000, max_pos=128)


@pytest.mark.parametrize("variant", [
    dict(weight_tier=1, ring_layers=1), dict(weight_tier=1, ring_layers=2), dict(weight_tier=1, ring_layers=3),
    dict(weight_tier=1, ring_layers=2, chunk_bytes=65536), dict(weight_tier=1, kv_tier=1),
    dict(weight_tier=0, kv_tier=1), dict(weight_tier=1, ring_layers=3, kv_tier=1, chunk_bytes=1 << 20),
    dict(weight_tier=1, flags=0)])
def test_tier_and_ring_invariance_bit_identical(variant):
    pipo = pipo_mod()
    prompt = synth.prompts(3, 20, SMALL.vocab)
    def syn(pl):
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 11)
        for j in range(SMALL.n_layers):
            pl.load_synthetic(j, 11)
    ref, _ = _run(pipo, SMALL, dict(weight_tier=pipo.PIPO_TIER_DEVICE), syn, prompt, 5)
    got, st = _run(pipo, SMALL, variant, syn, prompt, 5)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("shape,b,P,G,wfmt", [
    (synth.OPTShape(d_model=1024, n_layers=3, n_heads=16, ffn_dim=4096, vocab=2048, max_pos=256), 16, 48, 8, "int4"),
    (synth.OPTShape(d_model=1024, n_layers=2, n_heads=8, ffn_dim=4096, vocab=2048, max_pos=256), 20, 33, 8, "int4"),
    (synth.OPTShape(d_model=512, n_layers=2, n_heads=8, ffn_dim=2048, vocab=1500, max_pos=256), 6, 40, 8, "fp16"),
    (synth.OPTShape(d_model=512, n_layers=2, n_heads=4, ffn_dim=2048, vocab=1500, max_pos=256), 17, 24, 8, "fp16"),
])
def test_model_vs_oracle(shape, b, P, G, wfmt):
    pipo = pipo_mod()
    emb = synth.embed_masters(shape)
    layers = [synth.layer_masters(shape, j) for j in range(shape.n_layers)]
    ref = _oracle(shape, emb, layers, wfmt, P + G)
    cfg = pipo.make_config(shape, max_batch=b, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST,
                           wfmt=pipo.PIPO_W_INT4_G64 if wfmt == "int4" else pipo.PIPO_W_FP16)
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        res = teacher_forced(pl, ref, synth.prompts(b, P, shape.vocab), G)
    # every decided row's id is asserted equal inside teacher_forced(); the undecided
    # (near-tie) rows are capped at 2 % of all rows and reported
    assert_near_ties(res, b)


def test_api_errors():
    pipo = pipo_mod()
    cfg = pipo.make_config(SMALL, max_batch=2, max_seq=8, weight_tier=pipo.PIPO_TIER_HOST)
    with pipo.Pipeline(cfg) as pl:
        with pytest.raises(pipo.PipoError) as e:
            pl.decode_step(np.zeros(2, np.int32))
        assert e.value.status == pipo.PIPO_E_STATE
        with pytest.raises(pipo.PipoError) as e:
            pl.prefill(np.zeros((2, 4), np.int32))          # weights missing
        assert e.value.status == pipo.PIPO_E_STATE
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 1)
        for j in range(SMALL.n_layers):
            pl.load_synthetic(j, 1)
        with pytest.raises(pipo.PipoError) as e:
            pl.prefill(np.zeros((3, 4), np.int32))          # b > max_batch
        assert e.value.status == pipo.PIPO_E_INVALID_ARG
        with pytest.raises(pipo.PipoError) as e:
            pl.prefill(np.zeros((2, 8), np.int32))          # P >= max_seq
        assert e.value.status == pipo.PIPO_E_INVALID_ARG
        with pytest.raises(pipo.PipoError) as e:
            pl.prefill(np.full((2, 4), SMALL.vocab, np.int32))   # id out of range
        assert e.value.status == pipo.PIPO_E_INVALID_ARG
        nxt, _ = pl.prefill(np.zeros((2, 6), np.int32))
        nxt, _ = pl.decode_step(nxt)
        nxt, _ = pl.decode_step(nxt)
        with pytest.raises(pipo.PipoError) as e:
            pl.decode_step(nxt)                              # KV capacity exceeded
        assert e.value.status == pipo.PIPO_E_INVALID_ARG
    bad = pipo.make_config(SMALL, max_batch=2, max_seq=8)
    bad.d_model = 500
    with pytest.raises(pipo.PipoError) as e:
        pipo.pipeline_init(bad)
    assert e.value.status == pipo.PIPO_E_INVALID_ARG


def test_stats_busy_and_launches():
    pipo = pipo_mod()
    prompt = synth.prompts(4, 16, SMALL.vocab)
    def syn(pl):
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 3)
        for j in range(SMALL.n_layers):
            pl.load_synthetic(j, 3)
    _, st = _run(pipo, SMALL, dict(weight_tier=pipo.PIPO_TIER_HOST), syn, prompt, 6, want_logits=False)
    assert st["decode_steps"] == 5 and st["kernel_launches"] > 0
    for k in ("copy_busy", "kernel_busy", "union_busy"):
        assert 0 < st[k] <= 1.0 + 1e-6, (k, st[k])
    assert st["union_busy"] >= max(st["copy_busy"], st["kernel_busy"]) - 1e-9
    assert st["h2d_bytes"] > 0 and st["window_s"] > 0


@pytest.mark.parametrize("copy_us,comp_us,variant", [
    (400, 0, dict(weight_tier=1, ring_layers=2)), (0, 400, dict(weight_tier=1, ring_layers=2)),
    (300, 300, dict(weight_tier=1, ring_layers=1)), (250, 0, dict(weight_tier=1, ring_layers=3, chunk_bytes=1 << 16)),
    (300, 100, dict(weight_tier=1, ring_layers=2, kv_tier=1)), (0, 300, dict(weight_tier=0, kv_tier=1))])
def test_injected_delays_bit_identical(copy_us, comp_us, variant):
    """The method's invariance under timing (reading Q9): a slow host
    link (a busy wait before every layer's transfer on the copy stream) or slow compute
    (one before every layer's kernels) changes only when things happen, never the
    logits — the events order every consumer after its producer."""
    pipo = pipo_mod()
    prompt = synth.prompts(3, 20, SMALL.vocab)
    def syn(pl):
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 11)
        for j in range(SMALL.n_layers):
            pl.load_synthetic(j, 11)
    ref, _ = _run(pipo, SMALL, dict(weight_tier=pipo.PIPO_TIER_DEVICE), syn, prompt, 5)
    got, _ = _run(pipo, SMALL, variant, syn, prompt, 5,
                  hook=lambda pl: pipo.pipo_debug_inject(pl.ctx, copy_us, comp_us))
    assert np.array_equal(got, ref)


def _ring_checksum(blob):
    """SPEC.md:324's chunk checksum as pipo.h defines it: sum_i w_i * (2i + 1) mod 2^64
    over the blob's little-endian 64-bit words."""
    w = blob.view("<u8")
    return int(np.sum(w * (2 * np.arange(w.size, dtype=np.uint64) + 1), dtype=np.uint64))


@pytest.mark.parametrize("variant", [dict(ring_layers=2), dict(ring_layers=1, chunk_bytes=1 << 16),
                                     dict(ring_layers=3, chunk_bytes=(1 << 20) + 4096), dict(ring_layers=2, kv_tier=1)])
def test_ring_checksums_equal_host_blob(variant):
    """Every layer lands in its HBM ring slot byte for byte as the pinned host store
    holds it, for whole-blob and chunked transfers and all ring depths —
    checked by the GPU's checksum of the slot against numpy's of the host blob."""
    pipo = pipo_mod()
    prompt = synth.prompts(3, 20, SMALL.vocab)
    cfg = pipo.make_config(SMALL, max_batch=3, max_seq=25, weight_tier=pipo.PIPO_TIER_HOST, **variant)
    with pipo.Pipeline(cfg) as pl:
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 11)
        for j in range(SMALL.n_layers):
            pl.load_synthetic(j, 11)
        pipo.pipo_debug_inject(pl.ctx, 0, 0, True)
        nxt, _ = pl.prefill(prompt)
        for _ in range(3):
            nxt, _ = pl.decode_step(nxt)
        got = pipo.pipo_debug_ring_checksums(pl.ctx, SMALL.n_layers)
        want = [_ring_checksum(pipo.pipo_debug_read_blob(pl.ctx, j)) for j in range(SMALL.n_layers)]
    assert [int(x) for x in got] == want
    assert len(set(want)) == SMALL.n_layers          # the layers differ (the check is not vacuous)


@pytest.mark.parametrize("env_kw", [{}, {"PIPO_DISK_DELAY_US": "300"}])
def test_disk_tier_bit_identical(tmp_path, monkeypatch, env_kw):
    """DISK tier (blob files -> reader pool -> pinned ring -> H2D): same
    logits as the DEVICE tier, also with injected reader delays."""
    pipo = pipo_mod()
    for k, v in env_kw.items():
        monkeypatch.setenv(k, v)
    prompt = synth.prompts(3, 20, SMALL.vocab)
    def syn(pl):
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 11)
        for j in range(SMALL.n_layers):
            pl.load_synthetic(j, 11)
    ref, _ = _run(pipo, SMALL, dict(weight_tier=pipo.PIPO_TIER_DEVICE), syn, prompt, 5)
    got, st = _run(pipo, SMALL, dict(weight_tier=pipo.PIPO_TIER_DISK, disk_dir=str(tmp_path), chunk_bytes=1 << 18,
                                     disk_threads=3), syn, prompt, 5)
    assert np.array_equal(got, ref)
    assert len(list(tmp_path.glob("layer_*.pipo"))) == SMALL.n_layers


def test_disk_tier_io_failure_surfaces(tmp_path, monkeypatch):
    pipo = pipo_mod()
    monkeypatch.setenv("PIPO_DISK_FAIL_AT", "5")
    cfg = pipo.make_config(SMALL, max_batch=2, max_seq=16, weight_tier=pipo.PIPO_TIER_DISK, disk_dir=str(tmp_path),
                           chunk_bytes=1 << 18)
    with pipo.Pipeline(cfg) as pl:
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 1)
        for j in range(SMALL.n_layers):
            pl.load_synthetic(j, 1)
        with pytest.raises(pipo.PipoError) as e:
            pl.prefill(np.zeros((2, 4), np.int32))
        assert e.value.status == pipo.PIPO_E_IO
        with pytest.raises(pipo.PipoError) as e:       # poisoned afterwards
            pl.prefill(np.zeros((2, 4), np.int32))
        assert e.value.status == pipo.PIPO_E_STATE



@pytest.mark.parametrize("shape,b,P,G", [
    (synth.OPTShape(d_model=1024, n_layers=2, n_heads=8, ffn_dim=4096, vocab=2048, max_pos=256), 4, 40, 5),
    (synth.OPTShape(d_model=512, n_layers=2, n_heads=8, ffn_dim=2048, vocab=1500, max_pos=256), 20, 24, 4),
])
def test_int4_kv_cache_vs_oracle(shape, b, P, G):
    """NEXT-2: the INT4 KV cache against the oracle's int4-KV semantics."""
    pipo = pipo_mod()
    emb = synth.embed_masters(shape)
    layers = [synth.layer_masters(shape, j) for j in range(shape.n_layers)]
    ref = opt.OracleOPT.from_masters(shape.n_heads, emb, layers, "int4", P + G, kv_int4=True)
    for kv_tier in (pipo.PIPO_TIER_DEVICE, pipo.PIPO_TIER_HOST):
        cfg = pipo.make_config(shape, max_batch=b, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST,
                               kv_tier=kv_tier, kv_fmt=pipo.PIPO_W_INT4_G64)
        with pipo.Pipeline(cfg) as pl:
            load_masters(pl, emb, layers)
            ref.past = 0
            teacher_forced(pl, ref, synth.prompts(b, P, shape.vocab), G)


def test_int4_kv_tiers_bit_identical():
    pipo = pipo_mod()
    prompt = synth.prompts(3, 20, SMALL.vocab)
    def syn(pl):
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 5)
        for j in range(SMALL.n_layers):
            pl.load_synthetic(j, 5)
    ref, _ = _run(pipo, SMALL, dict(weight_tier=0, kv_fmt=1), syn, prompt, 5)
    for variant in (dict(weight_tier=1, kv_tier=1, kv_fmt=1), dict(weight_tier=1, kv_tier=1, kv_fmt=1, ring_layers=3),
                    dict(weight_tier=0, kv_tier=1, kv_fmt=1)):
        got, _ = _run(pipo, SMALL, variant, syn, prompt, 5)
        assert np.array_equal(got, ref)
    fp, _ = _run(pipo, SMALL, dict(weight_tier=0), syn, prompt, 5)
    assert np.array_equal(fp[0], ref[0])          # prefill attends over fresh fp16 K/V: identical
    assert not np.array_equal(fp[1:], ref[1:])    # decode reads the int4 cache


@pytest.mark.parametrize("kv_tier", [0, 1])
def test_int4_kv_decode_reads_own_row_quantized(kv_tier):
    """Reading Q17b on the GPU: on the hand-built model of tests/q17b_model.py the two
    readings of an int4 KV decode step differ by 0.063 per element; the pipeline's
    layer output must match reading A (own row read back from the int4 cache) to
    fp16 accuracy and be far from reading B (own row in full precision)."""
    from tests import q17b_model as qm
    pipo = pipo_mod()
    emb, layers = qm.masters()
    b = 2
    ref_a = opt.OracleOPT.from_masters(1, emb, layers, "int4", 4, kv_int4=True)
    ref_b = opt.OracleOPT.from_masters(1, emb, layers, "int4", 4, kv_int4=True)
    ref_a.prefill(qm.prompt(b))
    ref_a.decode(qm.decode_tokens(b))
    ref_b.prefill(qm.prompt(b))
    ref_b.kv_int4 = False                 # decode: own row fresh, old rows from the int4 cache
    ref_b.decode(qm.decode_tokens(b))
    want_a, want_b = ref_a.capture[0][:, 0], ref_b.capture[0][:, 0]
    cfg = pipo.make_config(qm.SHAPE, max_batch=b, max_seq=4, weight_tier=pipo.PIPO_TIER_HOST, kv_tier=kv_tier,
                           kv_fmt=pipo.PIPO_W_INT4_G64)
    with pipo.Pipeline(cfg) as pl:
        load_masters(pl, emb, layers)
        pl.prefill(qm.prompt(b))
        cap = np.zeros((1, b, 1, qm.SHAPE.d_model), np.float32)
        pipo.pipo_debug_capture(pl.ctx, cap)
        pl.decode_step(qm.decode_tokens(b))
    got = cap[0][:, 0].astype(np.float64)
    err_a = np.abs(got - want_a)[:, 1:].max()
    gap = np.abs(want_a - want_b)[:, 1:].min()
    assert gap > 0.05 and err_a < 5e-3, (err_a, gap)
    assert np.abs(got - want_b)[:, 1:].min() > 0.04
