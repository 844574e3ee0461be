"""CPU-side checks of the C-ABI library (no GPU needed).

* libpipo.so loads and exports every function include/pipo.h declares;
* pipeline_init fails loudly (PIPO_E_CUDA) when no device exists — there is no
  CPU fallback;
* the HOST quantizer behind load_layer_weights (pure C++) is bit-exact with the
  oracle's encoding (codes and fp16 scale bits), including its domain errors.
"""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import quant

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pipo():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_03664_b200 import pipo as p
    return p


def _declared():
    src = open(os.path.join(ROOT, "include", "pipo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:pipo_status|void\s*\*?|const char\s*\*|int32_t|int64_t)\s+(\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_exports_every_declared_symbol(pipo):
    names = _declared()
    assert "pipeline_init" in names and "decode_step" in names and len(names) >= 15
    lib = ctypes.CDLL(pipo.lib_path())
    for n in names:
        assert hasattr(lib, n), f"{n} declared in pipo.h but not exported"
    assert set(names) == set(pipo.EXPORTED)
    assert pipo.pipo_abi_version() == 5


def test_so_is_sm100a(pipo):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pipo.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", "x") != "x" and False, reason="")
def test_init_without_gpu_fails_loudly(pipo):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import pipo_synth as synth
    with pytest.raises(pipo.PipoError) as e:
        pipo.pipeline_init(pipo.make_config(synth.OPT_125M, max_batch=1, max_seq=8))
    assert e.value.status == pipo.PIPO_E_CUDA


@pytest.mark.parametrize("seed", [0, 1])
def test_host_quantizer_bit_exact(pipo, seed):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((130, 320)) * 0.02).astype(np.float16).astype(np.float32)
    w[3, :64] = 0                      # zero group
    w[4, :64] = 0.875                  # exact constant group
    w[5, :64] = 2.5e-7 * rng.standard_normal(64).astype(np.float32)   # subnormal scale
    w[6, 64:128] = rng.choice([-1, 1], 64) * 4095 * 2.0**-14          # rounding ties
    codes, scales = pipo.pipo_quantize_int4_g64(w)
    q, s = quant.quantize_int4_g64(w)
    assert np.array_equal(codes, quant.pack_int4(q))
    assert np.array_equal(scales, quant.scales_to_bits(s))


def test_host_quantizer_domain_errors(pipo):
    with pytest.raises(pipo.PipoError):
        pipo.pipo_quantize_int4_g64(np.full((1, 64), np.nan, dtype=np.float32))
    with pytest.raises(pipo.PipoError):
        pipo.pipo_quantize_int4_g64(np.full((1, 64), 1e6, dtype=np.float32))


def _write_blob_file(directory, layer, payload, magic=b"PIPOBLB1"):
    hdr = bytearray(4096)
    hdr[0:8] = magic
    hdr[8:12] = (1).to_bytes(4, "little")
    hdr[12:16] = layer.to_bytes(4, "little")
    hdr[16:24] = len(payload).to_bytes(8, "little")
    with open(os.path.join(directory, f"layer_{layer}.pipo"), "wb") as f:
        f.write(bytes(hdr) + payload.tobytes())


def test_disk_probe_reads_every_payload_byte(pipo, tmp_path):
    """The disk-tier roofline probe (pipo_probe_disk) reads exactly the
    payload of each layer file — ragged sizes, chunks smaller and larger than a file, more
    threads than chunks — checked by the position-weighted checksum computed here."""
    rng = np.random.default_rng(5)
    sizes = [10000, 8192, 123457, 1]
    want = 0
    for l, n in enumerate(sizes):
        b = rng.integers(0, 256, n, dtype=np.uint8)
        _write_blob_file(tmp_path, l, b)
        want += int((np.arange(1, n + 1, dtype=np.uint64) * b.astype(np.uint64)).sum(dtype=np.uint64))
    want %= 1 << 64
    for threads, chunk in [(1, 4096), (4, 8192), (8, 1 << 20)]:
        gbs, cs = pipo.pipo_probe_disk(str(tmp_path), len(sizes), threads, chunk, checksum=True)
        assert cs == want and gbs > 0
    gbs, cs = pipo.pipo_probe_disk(str(tmp_path), 2, 2, 4096)   # first two files only, no checksum
    assert cs is None and gbs > 0


def test_disk_probe_errors(pipo, tmp_path):
    _write_blob_file(tmp_path, 0, np.zeros(100, np.uint8))
    _write_blob_file(tmp_path, 1, np.zeros(100, np.uint8), magic=b"NOTABLOB")
    with pytest.raises(pipo.PipoError):                         # bad header
        pipo.pipo_probe_disk(str(tmp_path), 2, 1, 4096)
    with pytest.raises(pipo.PipoError):                         # missing file
        pipo.pipo_probe_disk(str(tmp_path / "none"), 1, 1, 4096)
    with pytest.raises(pipo.PipoError):                         # chunk not a 4 KiB multiple
        pipo.pipo_probe_disk(str(tmp_path), 1, 1, 5000)
    assert pipo.pipo_probe_disk(str(tmp_path), 1, 1, 4096)[0] > 0
