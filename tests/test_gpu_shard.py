"""NEXT-1 sharded weight streaming on one GPU: the 1-rank NCCL all-gather path runs the
whole sharded copy pipeline (padded ring slots, per-rank host store, in-place
all-gather on the copy stream, segment events after the gather) and must give
bit-identical logits to the plain host tier — the method's invariance (the transfer
path changes nothing).  Multi-rank runs need several GPUs (bench.py --shard-stream)."""
import numpy as np
import pytest

import pipo_synth as synth
from tests.gpu_util import load_masters, pipo_mod

pytestmark = pytest.mark.gpu

SMALL = synth.OPTShape(d_model=512, n_layers=4, n_heads=4, ffn_dim=2048, vocab=1000, max_pos=128)


def _run(pipo, shard, loader, kv_tier=0):
    prompt = synth.prompts(20, 12, SMALL.vocab)
    cfg = pipo.make_config(SMALL, max_batch=20, max_seq=16, weight_tier=pipo.PIPO_TIER_HOST, kv_tier=kv_tier)
    out = []
    with pipo.Pipeline(cfg) as pl:
        if shard:
            pipo.pipo_shard_stream_init(pl.ctx, 0, 1, pipo.pipo_nccl_unique_id())
        loader(pipo, pl)
        nxt, lg = pl.prefill(prompt, want_logits=True)
        out.append(lg)
        for _ in range(3):
            nxt, lg = pl.decode_step(nxt, want_logits=True)
            out.append(lg)
        st = pl.stats()
    return np.stack(out), st


def _masters(pipo, pl):
    load_masters(pl, synth.embed_masters(SMALL), [synth.layer_masters(SMALL, j) for j in range(SMALL.n_layers)])


def _synthetic(pipo, pl):
    pl.load_synthetic(pipo.PIPO_LAYER_EMBED, synth.WEIGHT_SEED)
    for j in range(SMALL.n_layers):
        pl.load_synthetic(j, synth.WEIGHT_SEED)


@pytest.mark.parametrize("loader", [_masters, _synthetic])
@pytest.mark.parametrize("kv_tier", [0, 1])
def test_sharded_stream_world1_bit_identical(loader, kv_tier):
    pipo = pipo_mod()
    base, _ = _run(pipo, False, loader, kv_tier)
    got, st = _run(pipo, True, loader, kv_tier)
    assert np.array_equal(base, got)
    assert st["h2d_bytes"] > 0


def test_shard_stream_init_errors():
    pipo = pipo_mod()
    cfg = pipo.make_config(SMALL, max_batch=2, max_seq=8, weight_tier=pipo.PIPO_TIER_DEVICE)
    with pipo.Pipeline(cfg) as pl:
        with pytest.raises(pipo.PipoError):
            pipo.pipo_shard_stream_init(pl.ctx, 0, 1, pipo.pipo_nccl_unique_id())   # not the HOST tier
    cfg = pipo.make_config(SMALL, max_batch=2, max_seq=8, weight_tier=pipo.PIPO_TIER_HOST)
    with pipo.Pipeline(cfg) as pl:
        pl.load_synthetic(0, synth.WEIGHT_SEED)
        with pytest.raises(pipo.PipoError):
            pipo.pipo_shard_stream_init(pl.ctx, 0, 1, pipo.pipo_nccl_unique_id())   # weights already loaded
        with pytest.raises(pipo.PipoError):
            pipo.pipo_shard_stream_init(pl.ctx, 2, 2, b"\0" * 128)                 # rank out of range
