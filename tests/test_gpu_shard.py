"""NEXT-1 sharded weight streaming on one GPU: the 1-rank NCCL all-gather path runs the
whole sharded copy pipeline (padded ring slots, per-rank host store, in-place
all-gather on the copy stream, segment events after the gather) and must give
bit-identical logits to the plain host tier — the method's invariance (the transfer
path changes nothing).  The peer transport (CUDA IPC, no NCCL) runs with two ranks as two
processes sharing this GPU: the N-rank path end to end on one device."""
import os

import numpy as np
import pytest

import pipo_synth as synth
from tests.gpu_util import load_masters, pipo_mod

pytestmark = pytest.mark.gpu

SMALL = synth.OPTShape(d_model=512, n_layers=4, n_heads=4, ffn_dim=2048, vocab=1000, max_pos=128)
B, P, G = 6, 12, 5            # per-rank batch, prompt, generated tokens (peer-transport tests)


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


# ---- N ranks through the peer transport (CUDA IPC + flags), 2 processes on one GPU ----
def _p2p_worker(rank, world, port, q, kw):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2504_03664_b200 import pipo
        from paper_2504_03664_b200.shard import shard_range
        cfg = pipo.make_config(SMALL, max_batch=B, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST, **kw)
        pl = pipo.Pipeline(cfg)
        h = pipo.pipo_shard_p2p_export(pl.ctx, rank, world)
        hs = [None] * world
        dist.all_gather_object(hs, h)
        pipo.pipo_shard_p2p_init(pl.ctx, hs)
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 13)
        for j in range(SMALL.n_layers):
            pl.load_synthetic(j, 13)
        lo, hi = shard_range(B * world, world, rank)
        prompt = synth.prompts(B * world, P, SMALL.vocab)[lo:hi]
        out = []
        nxt, lg = pl.prefill(prompt, want_logits=True)
        out.append(lg)
        for _ in range(G - 1):
            nxt, lg = pl.decode_step(nxt, want_logits=True)
            out.append(lg)
        st = pl.stats()
        dist.barrier()            # every peer is done reading this rank's ring
        pl.close()
        q.put((rank, np.stack(out), st["h2d_bytes"]))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kw", [dict(ring_layers=2), dict(ring_layers=3, kv_tier=1), dict(ring_layers=1)])
def test_p2p_sharded_two_ranks_bit_identical_to_one_gpu(kw):
    """NEXT-1 with two ranks (two processes sharing this GPU, peer copies through CUDA IPC):
    each rank streams half of every layer over the host link and pulls the other half
    from its peer's ring; every rank's logits equal, bit for bit, those of an unsharded
    single-GPU run on the same sequences (1 vs N GPUs on the same
    sequence), and each rank moved half the weight bytes over its link."""
    import torch.multiprocessing as mp
    pipo = pipo_mod()
    from paper_2504_03664_b200.shard import shard_range
    world = 2
    port = 31500 + os.getpid() % 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q, kw)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, lg, h2d = q.get(timeout=300)
        res[r] = (lg, h2d)
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r][0], str), res[r][0]
    plain = []
    for r in range(world):
        lo, hi = shard_range(B * world, world, r)
        prompt = synth.prompts(B * world, P, SMALL.vocab)[lo:hi]
        cfg = pipo.make_config(SMALL, max_batch=B, max_seq=P + G, weight_tier=pipo.PIPO_TIER_HOST, **kw)
        with pipo.Pipeline(cfg) as pl:
            pl.load_synthetic(pipo.PIPO_LAYER_EMBED, 13)
            for j in range(SMALL.n_layers):
                pl.load_synthetic(j, 13)
            out = []
            nxt, lg = pl.prefill(prompt, want_logits=True)
            out.append(lg)
            for _ in range(G - 1):
                nxt, lg = pl.decode_step(nxt, want_logits=True)
                out.append(lg)
            plain.append((np.stack(out), pl.stats()["h2d_bytes"]))
        assert np.array_equal(res[r][0], plain[r][0]), f"rank {r}"
        # weight bytes over this rank's link: about half (ids and, with host KV, the KV loads are per rank)
        if kw.get("kv_tier", 0) == 0:
            assert res[r][1] < 0.55 * plain[r][1], (res[r][1], plain[r][1])
