"""NEXT-3 on the GPU: the automatic configuration (Eq. (1)) applied
by pipeline_init (PIPO_F_AUTO_PLAN), the memory-efficient pipeline with host KV
(one layer's weights and KV resident, each KV save complete before
the slot is reused), and the runtime memory cross-check of SPEC.md:96: the context's
device occupancy never exceeds the App. B peak of the matching mode and is within 25 %
of it."""
import dataclasses

import numpy as np
import pytest

import pipo_synth as synth
from tests.gpu_util import pipo_mod

pytestmark = pytest.mark.gpu

# OPT-1.3B shapes (configs[1]) with 2 decoder layers: per-layer terms dominate the
# fixed workspace, so the App. B comparison is meaningful
SHAPE = dataclasses.replace(synth.OPT_1_3B, n_layers=2)
B, P, G = 16, 256, 16


def _spec(pipo):
    s = SHAPE
    return pipo.mem_spec(l=s.n_layers, d=s.d_model, V=s.vocab, h=s.n_heads, h_kv=s.n_heads, d_h=s.ffn_dim,
                         mlp_mats=2, p_weight=17 / 32, p_act=2.0)


def _run(pipo, cfg):
    prompt = synth.prompts(B, P, SHAPE.vocab)
    out = []
    with pipo.Pipeline(cfg) as pl:
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 21)
        for j in range(SHAPE.n_layers):
            pl.load_synthetic(j, 21)
        plan = pipo.pipo_get_plan(pl.ctx) if cfg.flags & pipo.PIPO_F_AUTO_PLAN else None
        nxt, lg = pl.prefill(prompt, want_logits=True)
        out.append(lg)
        for _ in range(3):
            nxt, lg = pl.decode_step(nxt, want_logits=True)
            out.append(lg)
        st = pl.stats()
    return np.stack(out), st, plan


def test_auto_plan_device_and_memory_efficient_host_kv():
    pipo = pipo_mod()
    s_max = P + G
    pre = pipo.pipo_memory_model(_spec(pipo), B, s_max, pipo.PIPO_STAGE_PREFILL, True)
    pre_np = pipo.pipo_memory_model(_spec(pipo), B, s_max, pipo.PIPO_STAGE_PREFILL, False)
    assert pre_np["m_peak"] < pre["m_peak"]
    ref, _, _ = _run(pipo, pipo.make_config(SHAPE, max_batch=B, max_seq=s_max, weight_tier=pipo.PIPO_TIER_DEVICE))

    # 1. plenty of HBM: Eq. (1) keeps everything on the GPU, performance-optimized pipeline
    got, st, plan = _run(pipo, pipo.make_config(SHAPE, max_batch=B, max_seq=s_max, flags=pipo.PIPO_F_AUTO_PLAN))
    assert plan["weight_tier"] == pipo.PIPO_TIER_DEVICE and plan["ring_layers"] == 2 and plan["block_bytes"] > 0
    assert np.array_equal(got, ref)

    # 2. M_GPU between the two App. B peaks: weights + KV on the host, memory-efficient
    #    pipeline (ring of one layer, one KV slot, saves serialised before the slot's reuse)
    budget = int((pre_np["m_peak"] + pre["m_peak"]) / 2)
    got, st, plan = _run(pipo, pipo.make_config(SHAPE, max_batch=B, max_seq=s_max, flags=pipo.PIPO_F_AUTO_PLAN,
                                                hbm_budget=budget))
    assert plan["weight_tier"] == pipo.PIPO_TIER_HOST and plan["ring_layers"] == 1, plan
    assert np.array_equal(got, ref)                     # the offloading changes nothing
    # SPEC.md:96 runtime cross-check against the no-preload (memory-efficient) peak
    assert st["hbm_bytes"] <= budget
    assert 0.75 * pre_np["m_peak"] <= st["hbm_bytes"] <= pre_np["m_peak"], (st["hbm_bytes"], pre_np["m_peak"])

    # 3. the performance-optimized host-KV pipeline against the preload peak
    got, st, _ = _run(pipo, pipo.make_config(SHAPE, max_batch=B, max_seq=s_max, weight_tier=pipo.PIPO_TIER_HOST,
                                             kv_tier=pipo.PIPO_TIER_HOST, ring_layers=2))
    assert np.array_equal(got, ref)
    assert 0.75 * pre["m_peak"] <= st["hbm_bytes"] <= pre["m_peak"], (st["hbm_bytes"], pre["m_peak"])

    # 4. a budget below even the memory-efficient peak is infeasible (Eq. (1), reading Q25)
    with pytest.raises(pipo.PipoError) as e:
        pipo.Pipeline(pipo.make_config(SHAPE, max_batch=B, max_seq=s_max, flags=pipo.PIPO_F_AUTO_PLAN,
                                       hbm_budget=int(pre_np["m_peak"] * 0.5)))
    assert e.value.status == pipo.PIPO_E_INFEASIBLE


@pytest.mark.parametrize("variant", [dict(weight_tier=1, kv_tier=1, ring_layers=1),
                                     dict(weight_tier=0, kv_tier=1, ring_layers=1),
                                     dict(weight_tier=1, kv_tier=1, ring_layers=1, kv_fmt=1)])
def test_memory_efficient_host_kv_bit_identical(variant):
    """R = 1 with the KV cache on the host (the memory-efficient pipeline)
    gives the same logits as the device tier, bit for bit, over prefill + decode."""
    pipo = pipo_mod()
    shape = synth.OPTShape(d_model=512, n_layers=4, n_heads=4, ffn_dim=2048, vocab=1000, max_pos=128)
    prompt = synth.prompts(3, 20, shape.vocab)

    def run(kw):
        cfg = pipo.make_config(shape, max_batch=3, max_seq=26, **kw)
        out = []
        with pipo.Pipeline(cfg) as pl:
            pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 11)
            for j in range(shape.n_layers):
                pl.load_synthetic(j, 11)
            nxt, lg = pl.prefill(prompt, want_logits=True)
            out.append(lg)
            for _ in range(5):
                nxt, lg = pl.decode_step(nxt, want_logits=True)
                out.append(lg)
        return np.stack(out)
    ref = run(dict(weight_tier=0, kv_fmt=variant.get("kv_fmt", 0)))
    assert np.array_equal(run(variant), ref)
