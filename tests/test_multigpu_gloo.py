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


# ---- NEXT-1 sharded weight streaming: host logic under a real 2-process collective ----
def test_shard_range_tiles_padded_blob():
    from paper_2504_03664_b200 import pipo
    for lb in (1, 4095, 4096, 3_780_096, 327_757_824, 115_900_416):
        for world in (1, 2, 3, 4, 8):
            spans = [pipo.pipo_shard_range(lb, world, r) for r in range(world)]
            S = spans[0][1]
            assert all(n == S for _, n in spans) and S % 4096 == 0
            assert [o for o, _ in spans] == [r * S for r in range(world)]
            assert lb <= S * world < lb + world * 4096          # padding < one 4 KiB page per rank
    with pytest.raises(pipo.PipoError):
        pipo.pipo_shard_range(100, 2, 2)


def _shard_worker(rank, world, port, q):
    """Emulates the copy stream of a sharded rank on CPU: stream own range, then the
    in-place all-gather (gloo standing in for NCCL over NVLink) must rebuild the blob."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_2504_03664_b200 import pipo
    lb = 3_780_096 + 123                                   # a c1 blob, not 4 KiB aligned
    off, S = pipo.pipo_shard_range(lb, world, rank)
    blob = np.zeros(S * world, dtype=np.uint8)
    blob[:lb] = np.random.default_rng(7).integers(0, 256, lb, dtype=np.uint8)   # same host store on every rank
    slot = torch.zeros(S * world, dtype=torch.uint8)
    slot[off:off + S] = torch.from_numpy(blob[off:off + S])                      # this rank's H2D range
    parts = [torch.zeros(S, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(parts, slot[off:off + S].clone())
    full = torch.cat(parts).numpy()
    q.put((rank, bool(np.array_equal(full, blob)), int(S)))
    dist.destroy_process_group()


def test_gloo_world2_sharded_stream_rebuilds_blob():
    world = 2
    port = 30500 + os.getpid() % 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)


# ---- bench.py launcher: `--gpus N` outside torchrun re-launches N ranks ----
def test_bench_metric_identical_in_both_arms():
    import bench
    for cfg in bench.CONFIGS:
        a = bench.parse(["--config", cfg])
        r = bench.parse(["--config", cfg, "--impl", "reference"])
        assert bench.metric_name(a) == bench.metric_name(r)
        assert bench.workload_config(a, 2) == bench.workload_config(r, 2)


def test_bench_self_launch_two_ranks_reference_arm():
    """`bench.py --gpus 2` (no WORLD_SIZE) re-runs itself under torch.distributed.run
    with 2 ranks over 127.0.0.1; rank 0 alone prints ONE line with n_gpus = 2 (the
    reference arm needs no GPU, so the launcher is exercised here on CPU)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--gpus", "2", "--steps", "2", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["steps"] * d["ms_per_step"] / 1e3 < 600       # the claimed timed work fits the run
