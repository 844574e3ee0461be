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
