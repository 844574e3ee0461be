"""GPU parity of the individual kernels through the C-ABI, against the oracle.

Bars (BASELINE.json north_star): bit-exact for the 4-bit pack/unpack (K8) and the
GPU quantizer; max relative error <= 2e-2 for the fp16/int4 linear layers and the
decode attention, with the special cases that pin layouts exactly.
"""
import numpy as np
import pytest

from oracle import opt, quant
from tests.gpu_util import pipo_mod, rel_inf

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    pipo = pipo_mod()
    import pipo_synth as synth
    shape = synth.OPTShape(d_model=256, n_layers=1, n_heads=4, ffn_dim=512, vocab=512, max_pos=64)
    pl = pipo.Pipeline(pipo.make_config(shape, max_batch=4, max_seq=16, weight_tier=pipo.PIPO_TIER_DEVICE))
    yield pipo, pl
    pl.close()


def test_unpack_exhaustive_bit_exact(env):
    pipo, pl = env
    scales = np.array([0.0999755859375, 2.0**-24, 3 * 2.0**-20, 6.103515625e-05, 1.0, 8188.0, 0.0, -0.5],
                      dtype=np.float16)
    packed = np.tile(np.arange(256, dtype=np.uint8), (len(scales), 1))          # K = 512
    s16 = np.repeat(scales[:, None], 8, axis=1)
    got = pipo.pipo_unpack_int4_g64(pl.ctx, packed, s16.view(np.uint16))
    ref = quant.unpack_scale_fp16(packed, s16)
    assert np.array_equal(got.view(np.uint16), ref.view(np.uint16))


@pytest.mark.parametrize("seed", [0, 1])
def test_gpu_quantizer_bit_exact(env, seed):
    pipo, pl = env
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((200, 384)) * 0.02).astype(np.float16).astype(np.float32)
    w[0, :64] = 0
    w[1, :64] = 0.875
    w[2, :64] = 2.5e-7 * rng.standard_normal(64).astype(np.float32)
    w[3, 64:128] = rng.choice([-1, 1], 64) * 4095 * 2.0**-14
    codes, scales = pipo.pipo_quantize_int4_g64_gpu(pl.ctx, w)
    q, s = quant.quantize_int4_g64(w)
    assert np.array_equal(codes, quant.pack_int4(q))
    assert np.array_equal(scales, quant.scales_to_bits(s))
    with pytest.raises(pipo.PipoError):
        pipo.pipo_quantize_int4_g64_gpu(pl.ctx, np.full((1, 64), np.inf, dtype=np.float32))


def _ref_linear(x16, w, bias, wfmt):
    wh = quant.quant_dequant(w) if wfmt == 1 else w.astype(np.float16).astype(np.float32)
    y = x16.astype(np.float64) @ wh.astype(np.float64).T
    if bias is not None:
        y = y + bias.astype(np.float16).astype(np.float64)
    return y


SHAPES = [(1, 128, 64), (3, 200, 256), (4, 384, 1024), (13, 130, 512), (16, 256, 256), (17, 384, 320),
          (40, 200, 1024), (64, 512, 2048), (100, 256, 192), (130, 384, 512), (300, 256, 320), (64, 7168, 7168), (1000, 640, 384),
          (512, 1152, 1024)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("wfmt", [1, 0])
def test_linear_vs_oracle(env, M, N, K, wfmt):
    pipo, pl = env
    rng = np.random.default_rng(M * 7 + N + K)
    x = rng.standard_normal((M, K)).astype(np.float16)
    w = (rng.standard_normal((N, K)) * 0.02).astype(np.float16).astype(np.float32)
    bias = (rng.uniform(-0.02, 0.02, N)).astype(np.float32)
    ref = _ref_linear(x, w, bias, wfmt)
    paths = [pipo.PATH_TC, pipo.PATH_GEMM] + ([pipo.PATH_GEMV] if wfmt == 1 and M <= 16 else []) + \
        ([pipo.PATH_WS] if wfmt == 1 and M <= 128 else []) + ([pipo.PATH_TM, pipo.PATH_PAIR] if wfmt == 1 and M <= 64 else []) + \
        ([pipo.PATH_TP] if wfmt == 1 else []) + ([pipo.PATH_STREAM, pipo.PATH_HEAD] if wfmt == 0 and M <= 64 else [])
    for path in paths:
        y = pipo.pipo_linear(pl.ctx, wfmt, path, x, w, bias)
        err = rel_inf(y, ref)
        assert err < 2e-2, (path, err)
        # fp16-rounded dequantized weights (GEMM) / exact codes (GEMV): far inside the bar
        assert err < (2e-3 if wfmt == 1 else 1e-4), (path, err)


@pytest.mark.parametrize("M,N,K", [(64, 512, 2048), (40, 200, 1024), (33, 384, 320), (64, 2304, 7168),
                                   (16, 1024, 8192), (64, 384, 4160), (1, 1664, 4096), (8, 7168, 28672),
                                   (64, 5376, 7168), (31, 896, 1088), (64, 12800, 2048), (48, 9984, 1536),
                                   (12, 4096, 1024), (24, 8192, 1024)])
@pytest.mark.parametrize("path", ["tm", "pair"])
def test_linear_tm_stream_k_deterministic(env, M, N, K, path):
    """The decode GEMMs (stream-K over CTAs / SM pairs; partials summed in k order by the
    reduce kernel or, for split tiles spanning <= ~3.5 CTAs, by the finishing CTA inside
    the kernel (tm: (40, 200, 1024), (31, 896, 1088), (64, 12800, 2048), (48, 9984, 1536)
    take the in-kernel fixup with 2-4 contributors per tile, as do (12, 4096, 1024) and
    (24, 8192, 1024) with the 16- and 32-token tiles), or by the finishing pair
    (pair)) within the bar
    and bit-reproducible run to run (the tier-invariance tests rely on it); K/64 odd
    (4160) takes the tm kernel's 1-k-block units; N not a multiple of 512 leaves the pair
    kernel's last quad of row-tiles partly empty."""
    pipo, pl = env
    p = pipo.PATH_TM if path == "tm" else pipo.PATH_PAIR
    rng = np.random.default_rng(M * 3 + N + K)
    x = rng.standard_normal((M, K)).astype(np.float16)
    w = (rng.standard_normal((N, K)) * 0.02).astype(np.float16).astype(np.float32)
    bias = (rng.uniform(-0.02, 0.02, N)).astype(np.float32)
    y = pipo.pipo_linear(pl.ctx, 1, p, x, w, bias)
    assert rel_inf(y, _ref_linear(x, w, bias, 1)) < 2e-3
    assert np.array_equal(y, pipo.pipo_linear(pl.ctx, 1, p, x, w, bias))


@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (97, 384, 320), (300, 640, 512), (1000, 1152, 256),
                                   (300, 128, 640), (700, 256, 2048)])
def test_linear_prefill_configs(env, M, N, K):
    """The prefill GEMM in both of its tile configurations (224-token tiles with two
    accumulators; 256-token tiles with one for the long-K case K >= 4N)."""
    pipo, pl = env
    rng = np.random.default_rng(M + N + K)
    x = rng.standard_normal((M, K)).astype(np.float16)
    w = (rng.standard_normal((N, K)) * 0.02).astype(np.float16).astype(np.float32)
    bias = (rng.uniform(-0.02, 0.02, N)).astype(np.float32)
    ref = _ref_linear(x, w, bias, 1)
    y = pipo.pipo_linear(pl.ctx, 1, pipo.PATH_TP, x, w, bias)
    assert rel_inf(y, ref) < 2e-3
    # one-hot rows -> dequantized columns exactly (fp16_rne(q*s) + bias, one rounding)
    q, s = quant.quantize_int4_g64(w)
    col = quant.dequantize(q, s).astype(np.float16).astype(np.float32)
    xo = np.zeros((M, K), np.float16)
    ks = np.arange(M) % K
    xo[np.arange(M), ks] = 1
    yo = pipo.pipo_linear(pl.ctx, 1, pipo.PATH_TP, xo, w, bias)
    b16 = bias.astype(np.float16).astype(np.float32)          # the library stores biases in fp16
    assert np.array_equal(yo, (col[:, ks].T + b16).astype(np.float32))


@pytest.mark.parametrize("path", ["gemv", "gemm", "tc", "ws", "tm", "tp", "pair"])
def test_linear_special_cases_exact(env, path):
    pipo, pl = env
    p = {"gemv": pipo.PATH_GEMV, "gemm": pipo.PATH_GEMM, "tc": pipo.PATH_TC, "ws": pipo.PATH_WS, "tm": pipo.PATH_TM,
         "tp": pipo.PATH_TP, "pair": pipo.PATH_PAIR}[path]
    rng = np.random.default_rng(5)
    N, K = 200, 256
    w = (rng.standard_normal((N, K)) * 0.02).astype(np.float16).astype(np.float32)
    bias = rng.uniform(-0.02, 0.02, N).astype(np.float16).astype(np.float32)
    # x = 0 -> bias exactly
    y0 = pipo.pipo_linear(pl.ctx, 1, p, np.zeros((3, K), np.float16), w, bias)
    assert np.array_equal(y0, np.broadcast_to(bias, (3, N)))
    # one-hot x_k -> column k of the dequantized weight (+ bias, one fp32 rounding):
    # GEMV multiplies exact codes: q*s exact; GEMM multiplies fp16_rne(q*s) (kernel K8)
    q, s = quant.quantize_int4_g64(w)
    col_exact = quant.dequantize(q, s)
    col_fp16 = col_exact.astype(np.float16).astype(np.float32)
    for k in (0, 63, 64, 255):
        x = np.zeros((2, K), np.float16)
        x[:, k] = 1
        y = pipo.pipo_linear(pl.ctx, 1, p, x, w, bias)
        col = col_exact[:, k] if path == "gemv" else col_fp16[:, k]
        assert np.array_equal(y[0], (col + bias).astype(np.float32)), k
    # power-of-two linearity, bit-exact
    x = rng.standard_normal((4, K)).astype(np.float16)
    y1 = pipo.pipo_linear(pl.ctx, 1, p, x, w, None)
    y2 = pipo.pipo_linear(pl.ctx, 1, p, (x.astype(np.float32) * 4).astype(np.float16), w, None)
    assert np.array_equal(y2, y1 * 4)


@pytest.mark.parametrize("b,L,d,H", [(1, 1, 128, 2), (2, 7, 256, 4), (3, 65, 256, 2), (4, 300, 512, 4),
                                     (2, 544, 1024, 8), (64, 40, 512, 8)])
@pytest.mark.parametrize("variant", [0, 1, 3])
def test_attention_decode_vs_oracle(env, b, L, d, H, variant):
    """variant 0 = the launcher's choice, 1 = lane-group kernel, 3 = one row per warp."""
    pipo, pl = env
    rng = np.random.default_rng(b * 1000 + L)
    q = (rng.standard_normal((b, d)) * (d // H) ** -0.5).astype(np.float16)
    k = rng.standard_normal((L, b, d)).astype(np.float16)
    v = rng.standard_normal((L, b, d)).astype(np.float16)
    o = pipo.pipo_attention_decode(pl.ctx, q, k, v, H, variant)
    ref = opt.attention(q.astype(np.float64)[:, None], k.astype(np.float64).transpose(1, 0, 2),
                        v.astype(np.float64).transpose(1, 0, 2), L - 1, H)[:, 0]
    assert rel_inf(o, ref) < 2e-2
    assert rel_inf(o, ref) < 5e-3


def test_attention_special_cases_exact(env):
    pipo, pl = env
    rng = np.random.default_rng(9)
    b, d, H = 2, 256, 2
    q = rng.standard_normal((b, d)).astype(np.float16)
    k = rng.standard_normal((1, b, d)).astype(np.float16)
    v = rng.standard_normal((1, b, d)).astype(np.float16)
    # one cached position: softmax of one logit is 1 -> output is the V row, exactly
    o = pipo.pipo_attention_decode(pl.ctx, q, k, v, H)
    assert np.array_equal(o, v[0].astype(np.float32))
    # all-equal keys -> mean of V (within fp16 output rounding)
    L = 33
    k2 = np.repeat(k, L, axis=0)
    v2 = rng.standard_normal((L, b, d)).astype(np.float16)
    o2 = pipo.pipo_attention_decode(pl.ctx, q, k2, v2, H)
    assert np.abs(o2 - v2.astype(np.float64).mean(0)).max() < 2e-3


@pytest.mark.parametrize("b,n,past,d,H", [(1, 5, 0, 128, 2), (2, 64, 0, 256, 2), (2, 100, 0, 512, 4),
                                          (3, 33, 7, 256, 4), (1, 130, 70, 1024, 8), (2, 512, 0, 512, 4),
                                          (2, 300, 200, 512, 4), (1, 384, 0, 256, 2), (2, 129, 0, 256, 4)])
@pytest.mark.parametrize("kernel", ["tcgen05", "cuda_cores", "mma_sync"])
def test_attention_prefill_vs_oracle(env, b, n, past, d, H, kernel):
    """Causal prefill attention against the fp64 definition: the tcgen05 kernel (key
    ranges <= 512; longer ones fall back), the legacy mma.sync kernel and the CUDA-core
    reference; ragged q-tiles (n = 5, 33, 100, 129, 130, 300) and past > 0."""
    pipo, pl = env
    cuda_cores = {"tcgen05": 0, "cuda_cores": 1, "mma_sync": 2}[kernel]
    rng = np.random.default_rng(n * 100 + past + d)
    q = (rng.standard_normal((b, n, d)) * (d // H) ** -0.5).astype(np.float16)
    L = past + n
    k = rng.standard_normal((L, b, d)).astype(np.float16)
    v = rng.standard_normal((L, b, d)).astype(np.float16)
    o = pipo.pipo_attention_prefill(pl.ctx, q, k, v, past, H, cuda_cores)
    ref = opt.attention(q.astype(np.float64), k.astype(np.float64).transpose(1, 0, 2),
                        v.astype(np.float64).transpose(1, 0, 2), past, H)
    assert rel_inf(o, ref) < 2e-2
    # P is rounded to fp16 before P.V on the tensor-core path
    assert rel_inf(o, ref) < (5e-3 if cuda_cores else 1e-2)


@pytest.mark.parametrize("hd", [64, 128])
def test_attention_prefill_tc_rescale_paths(env, hd):
    """The tcgen05 kernel's online softmax rescales O only when a key block's max exceeds
    the reference max by more than 2^8: keys growing along the positions force it for
    some query rows of a warp and not for others (the warp-collective TMEM rescale must
    then run with alpha = 1 on the rest), across 4 key blocks; checked against fp64."""
    pipo, pl = env
    rng = np.random.default_rng(hd)
    b, n, H = 2, 512, 2
    d = H * hd
    q = rng.standard_normal((b, n, d))
    q *= np.where(np.arange(n) % 3 == 0, 2.0, 0.25)[None, :, None]            # rows with / without rescales
    k = rng.standard_normal((n, b, d)) * (1.0 + np.arange(n) / 48.0)[:, None, None]
    q = (q * hd ** -0.5).astype(np.float16)
    k = k.astype(np.float16)
    v = rng.standard_normal((n, b, d)).astype(np.float16)
    ref = opt.attention(q.astype(np.float64), k.astype(np.float64).transpose(1, 0, 2),
                        v.astype(np.float64).transpose(1, 0, 2), 0, H)
    o = pipo.pipo_attention_prefill(pl.ctx, q, k, v, 0, H, 0)
    assert rel_inf(o, ref) < 1e-2


@pytest.mark.parametrize("path", ["stream", "head"])
@pytest.mark.parametrize("M", [1, 16, 33, 64])
def test_linear_fp16_stream_exact(env, path, M):
    """The streaming fp16 tcgen05 GEMM (LM head a13 / fp16 decode linears): x = 0 gives the
    bias exactly, one-hot rows give the fp16 weight column exactly (one fp32 rounding of
    w + b), power-of-two scaling is exact; ragged N (last 128-row tile partly padding) and
    M below the tile width (TMA zero-fill)."""
    pipo, pl = env
    p = pipo.PATH_STREAM if path == "stream" else pipo.PATH_HEAD
    rng = np.random.default_rng(M + 3)
    N, K = 300, 320
    w = (rng.standard_normal((N, K)) * 0.02).astype(np.float16).astype(np.float32)
    bias = rng.uniform(-0.02, 0.02, N).astype(np.float16).astype(np.float32)
    y0 = pipo.pipo_linear(pl.ctx, 0, p, np.zeros((M, K), np.float16), w, bias)
    assert np.array_equal(y0, np.broadcast_to(bias, (M, N)))
    x = np.zeros((M, K), np.float16)
    ks = (np.arange(M) * 37) % K
    x[np.arange(M), ks] = 1
    y = pipo.pipo_linear(pl.ctx, 0, p, x, w, bias)
    assert np.array_equal(y, (w[:, ks].T + bias).astype(np.float32))
    x = rng.standard_normal((M, K)).astype(np.float16)
    y1 = pipo.pipo_linear(pl.ctx, 0, p, x, w, None)
    y2 = pipo.pipo_linear(pl.ctx, 0, p, (x.astype(np.float32) * 4).astype(np.float16), w, None)
    assert np.array_equal(y2, y1 * 4)
    assert rel_inf(y1, x.astype(np.float64) @ w.astype(np.float64).T) < 1e-4
