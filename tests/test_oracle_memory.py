"""Pins of oracle/memory.py (the paper's memory model and Eq. (1)) to values fixed
outside the oracle: hand-evaluated worked examples (tests/golden/memory_model.json,
each cited), the paper's own model sizes, and structural
properties of the formulas."""
import json
import os
from fractions import Fraction as Fr

import pytest

from oracle import memory as mm

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "memory_model.json")))
TINY = mm.Spec(l=2, d=8, V=16, h=2, h_kv=1, d_h=24)


@pytest.mark.parametrize("case", GOLD["ffn_hidden_dim"])
def test_ffn_hidden_dim_worked_examples(case):
    assert mm.ffn_hidden_dim(case["d"], case["m"], case["gamma"]) == case["d_h"]


def test_tiny_spec_weights_kv_and_decode_peak():
    g = GOLD["tiny_weights"]
    w = mm.weight_sizes(TINY)
    for k in ("w_embed", "w_mha", "w_mlp", "w_total"):
        assert w[k] == g[k], k
    assert mm.kv_cache_size(TINY, 1, 4) == GOLD["tiny_kv"]["C"]
    r = mm.peak_memory(TINY, 1, 4, "decode", False)
    assert r["m_mlp"] == GOLD["tiny_decode_no_preload_m_mlp"]["m_mlp"]


@pytest.mark.parametrize("case", GOLD["paper_sizes"], ids=lambda c: c["model"])
def test_paper_model_sizes(case):
    d_h = case.get("d_h") or mm.ffn_hidden_dim(case["d"], case["m"], case["gamma"])
    sp = mm.Spec(l=case["l"], d=case["d"], V=case["V"], h=case["h"], h_kv=case["h_kv"], d_h=d_h,
                 p_w=Fr(case["p"]), mlp_mats=case["mlp_mats"])
    W = mm.weight_sizes(sp)["w_total"]
    assert case["lo"] <= W <= case["hi"], (case["model"], float(W))


def test_llama_gqa_term_is_appendix_b_form():
    """Q23: K and V are both h_kv/h wide — W_mha(h_kv = h) = p d (4d + 1), and halving
    h_kv removes exactly p d * d (half of K plus half of V)."""
    full = mm.Spec(l=1, d=64, V=10, h=8, h_kv=8, d_h=100)
    half = mm.Spec(l=1, d=64, V=10, h=8, h_kv=4, d_h=100)
    assert mm.weight_sizes(full)["w_mha"] == 2 * 64 * (4 * 64 + 1)
    assert mm.weight_sizes(full)["w_mha"] - mm.weight_sizes(half)["w_mha"] == 2 * 64 * 64


def test_int4_precision_is_payload_plus_scales():
    """int4-g64: 4 bits per weight + one fp16 scale per 64 -> 17/32 B, so W scales by 17/64 vs fp16."""
    sp16 = mm.Spec(l=3, d=128, V=50, h=2, h_kv=2, d_h=256)
    sp4 = mm.Spec(l=3, d=128, V=50, h=2, h_kv=2, d_h=256, p_w=mm.P_INT4_G64)
    assert mm.weight_sizes(sp4)["w_total"] * 64 == mm.weight_sizes(sp16)["w_total"] * 17


def test_kv_linear_in_b_and_s():
    assert mm.kv_cache_size(TINY, 2, 4) == 2 * mm.kv_cache_size(TINY, 1, 4)
    assert mm.kv_cache_size(TINY, 1, 8) == 2 * mm.kv_cache_size(TINY, 1, 4)
    assert mm.kv_cache_size(TINY, 1, 0) == 0


@pytest.mark.parametrize("stage", ["prefill", "decode"])
@pytest.mark.parametrize("preload", [True, False])
def test_peak_is_max_and_monotone(stage, preload):
    base = dict(l=4, d=64, V=100, h=4, h_kv=2, d_h=176)
    r = mm.peak_memory(mm.Spec(**base), 2, 16, stage, preload)
    assert r["m_peak"] == max(r["m_mha"], r["m_mlp"], r["m_embed"])
    for key, bump in (("d", 128), ("V", 200), ("l", 8), ("d_h", 352)):
        r2 = mm.peak_memory(mm.Spec(**{**base, key: bump}), 2, 16, stage, preload)
        assert r2["m_peak"] >= r["m_peak"], key
    assert mm.peak_memory(mm.Spec(**base), 4, 16, stage, preload)["m_peak"] >= r["m_peak"]
    assert mm.peak_memory(mm.Spec(**base), 2, 32, stage, preload)["m_peak"] >= r["m_peak"]


def test_prefill_preload_adds_exactly_one_layer_of_weights():
    """App. B prefill: with preloading M_mha gains W_mlp, M_mlp gains W_mha, and M_embed
    gains max(W_mha, W_embed) — the next layer's (or the head's) weights."""
    sp = mm.Spec(l=4, d=64, V=100, h=4, h_kv=2, d_h=176)
    a, b = mm.peak_memory(sp, 2, 16, "prefill", True), mm.peak_memory(sp, 2, 16, "prefill", False)
    assert a["m_mha"] - b["m_mha"] == a["w_mlp"]
    assert a["m_mlp"] - b["m_mlp"] == a["w_mha"]
    assert a["m_embed"] - b["m_embed"] == max(a["w_mha"], a["w_embed"])


def test_prefill_attention_term_is_quadratic_in_s():
    """M_attn = p b h s^2: the s^2 part of M_mha, isolated by finite differences."""
    sp = mm.Spec(l=1, d=64, V=10, h=4, h_kv=4, d_h=100)
    f = [mm.peak_memory(sp, 1, s, "prefill", False)["m_mha"] for s in (10, 11, 12)]
    assert f[2] - 2 * f[1] + f[0] == 2 * 2 * 4       # second difference of p*h*s^2 = 2*p*h


def test_eq1_decision_table():
    """Every branch of Eq. (1), hand-placed thresholds around W, C, M."""
    sp = mm.Spec(l=4, d=64, V=100, h=4, h_kv=4, d_h=176)
    b, s = 2, 16
    W = mm.weight_sizes(sp)["w_total"]
    C = mm.kv_cache_size(sp, b, s)
    M = mm.peak_memory(sp, b, s, "prefill", True)["m_peak"]
    M0 = mm.peak_memory(sp, b, s, "prefill", False)["m_peak"]
    assert M0 < M
    p = mm.choose_plan(sp, b, s, M_GPU=W + M + 1, M_CPU=1, B_GPU=1, B_SSD=2)
    assert (p["tier"], p["mode"]) == ("gpu", "performance")
    p = mm.choose_plan(sp, b, s, M_GPU=W + M, M_CPU=W + C + 1, B_GPU=2, B_SSD=1)
    assert (p["tier"], p["mode"]) == ("cpu", "performance")
    p = mm.choose_plan(sp, b, s, M_GPU=M, M_CPU=W + C + 1, B_GPU=2, B_SSD=1)
    assert (p["tier"], p["mode"]) == ("cpu", "memory_efficient")
    p = mm.choose_plan(sp, b, s, M_GPU=W + M, M_CPU=W + C, B_GPU=2, B_SSD=1)
    assert p["tier"] == "disk"
    p = mm.choose_plan(sp, b, s, M_GPU=W + M, M_CPU=W + C + 1, B_GPU=1, B_SSD=2)   # literal else-chain
    assert p["tier"] == "disk"
    with pytest.raises(ValueError):
        mm.choose_plan(sp, b, s, M_GPU=M0, M_CPU=1e18, B_GPU=2, B_SSD=1)


def test_quant_kernel_below_batch_16():
    """the INT4 kernel serves batch sizes less than 16."""
    sp = mm.Spec(l=1, d=64, V=10, h=4, h_kv=4, d_h=100, p_w=mm.P_INT4_G64)
    big = dict(M_GPU=1e18, M_CPU=1e18, B_GPU=2, B_SSD=1)
    assert mm.choose_plan(sp, 15, 8, **big)["use_quant_kernel"]
    assert not mm.choose_plan(sp, 16, 8, **big)["use_quant_kernel"]
    assert not mm.choose_plan(mm.Spec(l=1, d=64, V=10, h=4, h_kv=4, d_h=100), 4, 8, **big)["use_quant_kernel"]


def test_block_size_choice():
    """App. A: plateau at 32 MiB -> 32 MiB; one entry -> it; increasing -> the largest."""
    MiB = 1 << 20
    sizes = [1 * MiB, 8 * MiB, 32 * MiB, 128 * MiB]
    assert mm.choose_block_size(sizes, [10, 30, 50, 51]) == 32 * MiB
    assert mm.choose_block_size([8 * MiB], [3.0]) == 8 * MiB
    assert mm.choose_block_size(sizes, [1, 2, 3, 4]) == 128 * MiB
    # the disk edge bounds the pick (min over edges): disk best at 8 MiB, h2d flat
    assert mm.choose_block_size(sizes, [50, 50, 50, 50], [5, 9, 9.2, 9.3]) == 8 * MiB
