"""Host-side measurement logic of bench.py (no GPU): the CUPTI kernel-time accounting
behind the bench line's `roofline` object and the roofline fraction itself."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

CLASSES = {"linear_decode": ("gemm_tm_kernel", "ws_reduce"), "attn_decode": ("attn_decode",)}


def test_exclusive_time_removes_pdl_overlap():
    # one stream: GEMM [0, 40], its reduce launched early [30, 47], attention launched early
    # [45, 200] (it waits for the reduce), a copy-engine transfer overlapping everything
    ev = [(7, 0.0, 40.0, "void pipo::gemm_tm_kernel<64>(...)"),
          (7, 30.0, 47.0, "void pipo::ws_reduce2_kernel<64, 1>(...)"),
          (7, 45.0, 200.0, "void pipo::attn_decode_kernel<128, 1>(...)"),
          (9, 0.0, 500.0, "Memcpy HtoD (Pinned -> Device)")]
    tot, names, n_streams = bench.exclusive_class_times(ev, CLASSES)
    assert n_streams == 1                                  # the memcpy is not a kernel
    assert tot["linear_decode"] == pytest.approx(47e-6)    # 40 + (47 - 40), not 40 + 17
    assert tot["attn_decode"] == pytest.approx(153e-6)     # 200 - 47, not 155
    assert names["linear_decode"] == {"void pipo::gemm_tm_kernel", "void pipo::ws_reduce2_kernel"}


def test_exclusive_time_streams_are_independent_and_gaps_are_not_counted():
    ev = [(1, 0.0, 10.0, "gemm_tm_kernel"), (1, 15.0, 20.0, "gemm_tm_kernel"),   # 5 us gap: idle, not counted
          (2, 5.0, 12.0, "attn_decode_kernel")]                                 # another stream overlaps freely
    tot, _, n = bench.exclusive_class_times(ev, CLASSES)
    assert n == 2
    assert tot["linear_decode"] == pytest.approx(15e-6)
    assert tot["attn_decode"] == pytest.approx(7e-6)


def test_kernel_fully_inside_predecessor_counts_zero():
    ev = [(1, 0.0, 100.0, "attn_decode_kernel"), (1, 10.0, 50.0, "ws_reduce2_kernel")]
    tot, _, _ = bench.exclusive_class_times(ev, CLASSES)
    assert tot["attn_decode"] == pytest.approx(100e-6)
    assert tot["linear_decode"] == 0.0


def test_roofline_picks_the_largest_class_and_the_binding_bound():
    peaks = {"hbm_gbs": 6500.0, "bf16_tflops_sustained": 1400.0}
    # linear: 87 MB + 19.7 GFLOP per unit -> tensor-bound (14.1 us) over HBM (13.4 us)
    cupti = {"linear_decode": {"us_per_unit": 37.0, "ms_per_step": 7.1, "bytes_per_unit": 87e6, "flops_per_unit": 19.73e9},
             "attn_decode": {"us_per_unit": 161.0, "ms_per_step": 7.7, "bytes_per_unit": 969e6, "flops_per_unit": 0.96e9}}
    r = bench.roofline_of(cupti, {}, {}, 10, peaks)
    assert r["kernel"] == "attn_decode" and r["bound"] == "hbm"
    assert r["frac"] == pytest.approx(969e6 / 6500e9 / 161e-6)
    lin = r["by_class"]["linear_decode"]
    assert lin["bound"] == "tensor"
    assert lin["frac"] == pytest.approx(19.73e9 / 1400e12 / 37e-6)
