"""The seeded input generator (pipo_synth): determinism, shapes and distributions
(SURVEY.md §8(d) recipe).  No method arithmetic lives there."""
import numpy as np

import pipo_synth as synth


def test_deterministic_and_fp16_exact():
    a = synth.draw(2504, 3, synth.T_W_QKV, synth.KIND_NORMAL, 0.02, 1000, 5000)
    b = synth.draw(2504, 3, synth.T_W_QKV, synth.KIND_NORMAL, 0.02, 1000, 5000)
    assert np.array_equal(a, b)
    assert np.array_equal(a.astype(np.float16).astype(np.float32), a)
    c = synth.draw(2504, 4, synth.T_W_QKV, synth.KIND_NORMAL, 0.02, 1000, 5000)
    assert not np.array_equal(a, c)


def test_draw_rows_matches_draw():
    full = synth.draw(7, 2, 8, synth.KIND_NORMAL, 0.02, 0, 10 * 64).reshape(10, 64)
    rows = synth.draw_rows(7, 2, 8, synth.KIND_NORMAL, 0.02, 64, [3, 7])
    assert np.array_equal(rows, full[[3, 7]])


def test_distributions():
    n = 1 << 20
    w = synth.draw(1, 1, 2, synth.KIND_NORMAL, 0.02, 0, n)
    assert abs(w.std() - 0.02) < 2e-4 and abs(w.mean()) < 2e-4
    u = synth.draw(1, 1, 3, synth.KIND_UNIFORM, 0.02, 0, n)
    lim = 0.02 * (1 + 2.0**-10)   # fp16 rounding of the bound
    assert u.min() >= -lim and u.max() <= lim and abs(u.std() - 0.02 / np.sqrt(3)) < 2e-4
    g = synth.draw(1, 1, 0, synth.KIND_GAMMA, 0.1, 0, n)
    assert g.min() >= 0.9 - 1e-3 and g.max() <= 1.1 + 1e-3   # fp16 grid near 1 is 2^-11


def test_prompts_range():
    p = synth.prompts(16, 256, 50272)
    assert p.shape == (16, 256) and p.dtype == np.int32
    assert p.min() >= 4 and p.max() < 50272
    assert np.array_equal(p, synth.prompts(16, 256, 50272))


def test_llama_shapes_and_streams():
    """LLaMA3.1 tensor set (NEXT-4): shapes from the public 8B config, and the streams
    that share a role with OPT use the same tensor ids (so e.g. w_qkv rows of an 8B
    layer are the same counter stream as any other matrix in that slot)."""
    s = synth.LLAMA31_8B
    assert (s.head_dim, s.d_kv) == (128, 1024)
    spec = synth.llama_layer_tensor_specs(s)
    assert spec["w_qkv"][3] == (4096 + 2 * 1024, 4096)
    assert spec["w_fc1"][3] == (2 * 14336, 4096) and spec["w_fc2"][3] == (4096, 14336)
    assert set(spec) == {"ln1_g", "w_qkv", "w_out", "ln2_g", "w_fc1", "w_fc2"}     # no biases
    emb = synth.llama_embed_tensor_specs(s)
    assert emb["lm_head"][0] == synth.T_LM_HEAD and emb["lm_head"][3] == (128256, 4096)
    tiny = synth.LlamaShape(64, 1, 4, 2, 128, vocab=256, max_pos=64)
    m = synth.llama_layer_masters(tiny, 0)
    ref = synth.draw(synth.WEIGHT_SEED, 1, synth.T_W_QKV, synth.KIND_NORMAL, 0.02, 0, 128 * 64).reshape(128, 64)
    assert np.array_equal(m["w_qkv"], ref)
    assert np.all(np.abs(m["ln1_g"] - 1.0) <= 0.1 + 1e-3)
