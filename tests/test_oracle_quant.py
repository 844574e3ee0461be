"""Pins for oracle/quant.py against what the definition fixes (not against itself).

The int4-g64 encoding is
checked by hand-derived worked groups, exhaustive enumeration, and invariants a
plausible mistake would break (wrong rounding mode, unrounded scale, swapped
nibbles, wrong sign extension, wrong group axis).
"""
import numpy as np
import pytest

from oracle import quant


def _group(vals):
    g = np.zeros(64, dtype=np.float32)
    g[: len(vals)] = np.asarray(vals, dtype=np.float32)
    return g


def test_worked_group_a_hand_derived():
    # a = 0.7f; a/7 in fp32 = 0.100000001490116 (nearest fp32 to 0.09999999830);
    # fp16 grid in [1/16, 1/8) has step 2^-14: 0.1/2^-14 = 1638.4 -> 1638*2^-14
    #   s = 0.0999755859375 = fp16 bits 0x2E66 (exp 11, mantissa 614).
    # 0.7f/s = 7.0017 -> 7 ; -0.35f/s = -3.50085 -> -4 ; 0.1f/s = 1.00024 -> 1
    # 0.05f/s = 0.50012 -> 1  (an UNROUNDED scale 0.1 would give rint(0.5)=0)
    # 4095*2^-14 / s = 2.5 exactly -> 2 (half-to-even; half-away would give 3)
    # 5733*2^-14 / s = 3.5 exactly -> 4 (half-to-even)
    vals = [0.7, -0.35, 0.1, 0.0, 0.05, 4095 * 2.0**-14, -4095 * 2.0**-14, 5733 * 2.0**-14]
    w = _group(vals)[None, :]
    q, s = quant.quantize_int4_g64(w)
    assert quant.scales_to_bits(s)[0, 0] == 0x2E66
    assert q[0, :8].tolist() == [7, -4, 1, 0, 1, 2, -2, 4]
    assert np.all(q[0, 8:] == 0)
    packed = quant.pack_int4(q)
    # byte0 = 7 | (-4 & 15) << 4 = 0xC7 ; byte1 = 1 | 0 ; byte2 = 1 | 2 << 4 ; byte3 = (-2 & 15) | 4 << 4
    assert packed[0, :4].tolist() == [0xC7, 0x01, 0x21, 0x4E]
    wh = quant.dequantize(q, s)
    assert wh[0, 0] == np.float32(7 * 1638 * 2.0**-14)


def test_worked_group_negative_absmax():
    # a = 1.0; 1/7 (fp32) = 0.142857149; fp16 step in [1/8,1/4) is 2^-13:
    # 0.142857149/2^-13 = 1170.29 -> 1170*2^-13 = 0.142822265625, bits 12<<10|146 = 0x3092.
    # -1/s = -7.0017 -> -7 ; 0.5/s = 3.50085 -> 4 ; byte = (-7 & 15) | 4 << 4 = 0x49
    w = _group([-1.0, 0.5])[None, :]
    q, s = quant.quantize_int4_g64(w)
    assert quant.scales_to_bits(s)[0, 0] == 0x3092
    assert q[0, :2].tolist() == [-7, 4]
    assert quant.pack_int4(q)[0, 0] == 0x49


def test_zero_and_constant_groups():
    w = np.zeros((2, 128), dtype=np.float32)
    w[1, :64] = 0.875          # 7 * 0.125: a/7 = 0.125 exactly -> exact dequant
    w[1, 64:] = -0.3           # constant but not exactly representable: codes all equal
    q, s = quant.quantize_int4_g64(w)
    assert np.all(q[0] == 0) and np.all(quant.scales_to_bits(s)[0] == 0)
    assert np.all(q[1, :64] == 7) and quant.scales_to_bits(s)[1, 0] == 0x3000
    assert np.all(quant.dequantize(q, s)[1, :64] == np.float32(0.875))
    assert np.all(q[1, 64:] == q[1, 64])


def test_group_axis_is_k():
    # groups are 64 consecutive elements along K within a row, never across rows
    w = np.zeros((2, 128), dtype=np.float32)
    w[0, 0] = 1.0      # group (0,0)
    w[0, 64] = 0.01    # group (0,1) must get its own small scale
    w[1, 0] = 0.5
    q, s = quant.quantize_int4_g64(w)
    s32 = s.astype(np.float32)
    assert s32[0, 1] < 0.01 and s32[0, 0] > 0.1
    assert q[0, 64] == 7 and q[0, 0] == 7 and q[1, 0] == 7


def test_exhaustive_pack_unpack_bijection():
    allbytes = np.arange(256, dtype=np.uint8)[None, :]
    codes = quant.unpack_int4(allbytes)
    assert codes.min() == -8 and codes.max() == 7
    # independent decode of every byte with Python ints
    for v in range(256):
        lo, hi = v & 15, v >> 4
        lo = lo - 16 if lo >= 8 else lo
        hi = hi - 16 if hi >= 8 else hi
        assert codes[0, 2 * v] == lo and codes[0, 2 * v + 1] == hi
    assert np.array_equal(quant.pack_int4(codes), allbytes)


def test_exhaustive_unpack_scale_fp16():
    # K8 contract: fp16_rne(q*s); checked with Python double arithmetic (q*s exact
    # in double, so float16() rounds once) over every byte x a scale set that
    # includes normal, subnormal and max-finite fp16 scales.
    scales = np.array([0.0999755859375, 2.0**-24, 3 * 2.0**-20, 6.103515625e-05,
                       1.0, 65504.0 / 8, 0.0], dtype=np.float16)
    packed = np.tile(np.arange(256, dtype=np.uint8), (len(scales), 1))   # [7, 256] -> K=512
    s16 = np.repeat(scales[:, None], 512 // 64, axis=1)
    out = quant.unpack_scale_fp16(packed, s16)
    for r, sc in enumerate(scales):
        for v in range(256):
            for j, nib in enumerate((v & 15, v >> 4)):
                qv = nib - 16 if nib >= 8 else nib
                ref = np.float16(qv * float(sc))
                got = out[r, 2 * v + j]
                assert got.view(np.uint16) == ref.view(np.uint16) or (ref == 0 and got == 0)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_invariants_random(seed):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((64, 512)) * 0.02).astype(np.float16).astype(np.float32)
    q, s = quant.quantize_int4_g64(w)
    s32 = np.repeat(s.astype(np.float32), 64, axis=1)
    wh = quant.dequantize(q, s)
    # |w - w_hat| <= s/2 elementwise
    assert np.all(np.abs(w - wh) <= s32 / 2)
    # normal scales never produce -8; absmax element maps to +-7
    assert q.min() >= -7 and q.max() <= 7
    g = w.reshape(64, 8, 64)
    am = np.argmax(np.abs(g), axis=2)
    qa = np.take_along_axis(q.reshape(64, 8, 64), am[..., None], 2)[..., 0]
    assert np.all(np.abs(qa) == 7)
    # idempotence: quantize(dequantize(quantize(w))) == quantize(w)
    q2, s2 = quant.quantize_int4_g64(wh)
    assert np.array_equal(q2, q) and np.array_equal(s2.view(np.uint16), s.view(np.uint16))
    # sign symmetry
    q3, s3 = quant.quantize_int4_g64(-w)
    assert np.array_equal(q3, -q) and np.array_equal(s3.view(np.uint16), s.view(np.uint16))
    # power-of-two scaling: codes equal, scale x 2^k (normal range)
    for k in (-3, 4):
        q4, s4 = quant.quantize_int4_g64(w * np.float32(2.0**k))
        assert np.array_equal(q4, q)
        assert np.array_equal(s4.astype(np.float32), s.astype(np.float32) * np.float32(2.0**k))


def test_subnormal_scale_clamps():
    # a/7 below fp16 min normal: the fp16 scale is subnormal and may round DOWN so far
    # that g/s exceeds 7.5; the clamp keeps codes in [-8, 7].
    w = _group([2.5e-7, -2.4e-7, 1e-7])[None, :]
    q, s = quant.quantize_int4_g64(w)
    assert q.min() >= -8 and q.max() <= 7
    assert s.astype(np.float32)[0, 0] > 0


def test_domain_errors():
    with pytest.raises(ValueError):
        quant.quantize_int4_g64(np.full((1, 64), np.inf, dtype=np.float32))
    with pytest.raises(ValueError):
        quant.quantize_int4_g64(np.full((1, 64), 1e6, dtype=np.float32))
    with pytest.raises(ValueError):
        quant.quantize_int4_g64(np.zeros((1, 65), dtype=np.float32))
