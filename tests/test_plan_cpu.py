"""The library's automatic-configuration calls (host C++, no GPU) against the oracle
(oracle/memory.py): memory model values bit-exact, Eq. (1) decisions identical,
block-size pick identical, error statuses."""
import numpy as np
import pytest

from oracle import memory as mm


@pytest.fixture(scope="module")
def pipo():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_03664_b200 import pipo as p
    return p


def _rand_spec(rng):
    h = int(rng.choice([1, 2, 4, 8, 12, 32, 40, 56]))
    group = int(rng.choice([g for g in (1, 2, 4, 8) if h % g == 0]))
    hd = int(rng.choice([16, 64, 128]))
    return mm.Spec(l=int(rng.integers(1, 100)), d=h * hd, V=int(rng.integers(1, 200000)), h=h, h_kv=h // group,
                   d_h=int(rng.integers(1, 60000)), p_w=[mm.P_FP16, mm.P_INT4_G64][int(rng.integers(2))],
                   p_a=mm.P_FP16, mlp_mats=int(rng.choice([2, 3])))


def _c_spec(pipo, sp):
    return pipo.mem_spec(l=sp.l, d=sp.d, V=sp.V, h=sp.h, h_kv=sp.h_kv, d_h=sp.d_h, mlp_mats=sp.mlp_mats,
                         p_weight=float(sp.p_w), p_act=float(sp.p_a))


def test_ffn_hidden_dim(pipo):
    for d, m, g in [(4096, 1024, 1.3), (3, 1, 1.0), (8, 4, 1.0), (8192, 1024, 1.3), (16384, 4096, 1.2)]:
        assert pipo.pipo_ffn_hidden_dim(d, m, g) == mm.ffn_hidden_dim(d, m, g)
    assert pipo.pipo_ffn_hidden_dim(0, 1, 1.0) == -1


@pytest.mark.parametrize("seed", range(4))
def test_memory_model_bit_exact(pipo, seed):
    rng = np.random.default_rng(seed)
    for _ in range(50):
        sp = _rand_spec(rng)
        b, s = int(rng.integers(1, 256)), int(rng.integers(0, 8192))
        for stage, sname in ((pipo.PIPO_STAGE_PREFILL, "prefill"), (pipo.PIPO_STAGE_DECODE, "decode")):
            for pre in (True, False):
                got = pipo.pipo_memory_model(_c_spec(pipo, sp), b, s, stage, pre)
                ref = mm.peak_memory(sp, b, s, sname, pre)
                for k, v in got.items():
                    assert v == float(ref[k]), (k, sp, b, s, sname, pre)


@pytest.mark.parametrize("seed", range(3))
def test_choose_plan_matches_oracle(pipo, seed):
    rng = np.random.default_rng(100 + seed)
    seen = set()
    for _ in range(300):
        sp = _rand_spec(rng)
        b, s = int(rng.integers(1, 64)), int(rng.integers(1, 4096))
        W = float(mm.weight_sizes(sp)["w_total"])
        M = float(mm.peak_memory(sp, b, s, "prefill", True)["m_peak"])
        hw = dict(m_gpu=float(M * rng.uniform(0.5, 3.0) + W * rng.uniform(0, 1.5)),
                  m_cpu=float(W * rng.uniform(0.5, 2.0)), b_gpu=float(rng.uniform(1, 64)), b_ssd=float(rng.uniform(1, 64)))
        try:
            ref = mm.choose_plan(sp, b, s, M_GPU=hw["m_gpu"], M_CPU=hw["m_cpu"], B_GPU=hw["b_gpu"], B_SSD=hw["b_ssd"])
        except ValueError:
            with pytest.raises(pipo.PipoError) as e:
                pipo.pipo_choose_plan(_c_spec(pipo, sp), b, s, **hw)
            assert e.value.status == pipo.PIPO_E_INFEASIBLE
            seen.add("infeasible")
            continue
        got = pipo.pipo_choose_plan(_c_spec(pipo, sp), b, s, **hw)
        tier = {"gpu": pipo.PIPO_TIER_DEVICE, "cpu": pipo.PIPO_TIER_HOST, "disk": pipo.PIPO_TIER_DISK}[ref["tier"]]
        assert got["weight_tier"] == tier
        assert got["ring_layers"] == (2 if ref["mode"] == "performance" else 1)
        assert got["use_quant_kernel"] == int(ref["use_quant_kernel"])
        assert (got["w_total"], got["c_total"], got["m_peak"]) == (float(ref["W"]), float(ref["C"]), float(ref["M"]))
        seen.add((ref["tier"], ref["mode"]))
    assert len(seen) >= 4, seen     # the random draw reaches most cells of the decision table


def test_block_size(pipo):
    MiB = 1 << 20
    sizes = [1 * MiB, 8 * MiB, 32 * MiB, 128 * MiB]
    for h2d, disk in [([10, 30, 50, 51], None), ([1, 2, 3, 4], None), ([50, 50, 50, 50], [5, 9, 9.2, 9.3])]:
        assert pipo.pipo_choose_block_size(sizes, h2d, disk) == mm.choose_block_size(sizes, h2d, disk)
    p = pipo.pipo_choose_plan(pipo.mem_spec(l=1, d=64, V=10, h=4, h_kv=4, d_h=100), 1, 8, m_gpu=1e12, m_cpu=1e12,
                              b_gpu=2, b_ssd=1, sizes=sizes, h2d_bps=[10, 30, 50, 51])
    assert p["block_bytes"] == 32 * MiB


def test_bad_arguments(pipo):
    with pytest.raises(pipo.PipoError) as e:
        pipo.pipo_memory_model(pipo.mem_spec(l=1, d=64, V=10, h=4, h_kv=3, d_h=100), 1, 1, 0, True)
    assert e.value.status == pipo.PIPO_E_INVALID_ARG
    with pytest.raises(pipo.PipoError):
        pipo.pipo_memory_model(pipo.mem_spec(l=0, d=64, V=10, h=4, h_kv=4, d_h=100), 1, 1, 0, True)
    with pytest.raises(pipo.PipoError):
        pipo.pipo_choose_plan(pipo.mem_spec(l=1, d=64, V=10, h=4, h_kv=4, d_h=100), 1, 8, m_gpu=0, m_cpu=1,
                              b_gpu=1, b_ssd=1)


def test_opt_configs_on_b200(pipo):
    """Reading Q19: on a 180 GB B200 Eq. (1) puts every benchmark config's weights on the
    GPU; the configs force the host / disk tier to exercise the streaming path."""
    import pipo_synth as synth
    for shape, b, s in [(synth.OPT_1_3B, 16, 288), (synth.OPT_6_7B, 32, 544), (synth.OPT_13B, 64, 544),
                        (synth.OPT_30B, 64, 544)]:
        sp = pipo.mem_spec(l=shape.n_layers, d=shape.d_model, V=shape.vocab, h=shape.n_heads, h_kv=shape.n_heads,
                           d_h=shape.ffn_dim, mlp_mats=2, p_weight=17 / 32, p_act=2.0)
        p = pipo.pipo_choose_plan(sp, b, s, m_gpu=180e9, m_cpu=190e9, b_gpu=55.6e9, b_ssd=5.3e9)
        assert p["weight_tier"] == pipo.PIPO_TIER_DEVICE and p["ring_layers"] == 2
