"""Multi-process (gloo, world_size 2, CPU) checks of the batch-shard host logic:
shard ranges partition the global batch, the timing reduction is a max over
ranks, and each rank's prompts are exactly its slice of the global prompt batch
(so N-GPU tokens equal the 1-GPU tokens on the same sequences)."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_03664_b200.shard import aggregate_throughput, max_over_ranks, shard_range


def test_shard_range_partitions():
    for gb in (64, 65, 128, 7):
        for world in (1, 2, 3, 4, 7):
            if gb < world:
                continue
            spans = [shard_range(gb, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == gb
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and b > a
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(1, 2, 0)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import pipo_synth as synth
    t = 1.0 + rank * 0.5                      # rank 1 is slower
    mx = max_over_ranks(t)
    lo, hi = shard_range(128, world, rank)
    mine = synth.prompts(128, 16, 1000)[lo:hi]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    dist.barrier()
    q.put((rank, mx, np.concatenate(gathered)))
    dist.destroy_process_group()


def test_gloo_world2_max_and_shards():
    world = 2
    port = 29500 + os.getpid() % 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import pipo_synth as synth
    full = synth.prompts(128, 16, 1000)
    for rank, mx, allp in res:
        assert mx == 1.5
        assert np.array_equal(allp, full)
    assert aggregate_throughput(64, 2, 10, 2.0) == 640.0
