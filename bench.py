"""bench.py — decode tokens/s of the streamed-weight PIPO pipeline (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--wfmt int4|fp16]
    python bench.py --impl reference ...     # the CPU oracle arm (reads oracle/)

A "step" is one decode_step: all n_layers decoder layers (weights streamed from
pinned host memory over PCIe, chunk by chunk, consumed as they land) plus the LM
head and greedy argmax, for a batch of b sequences per GPU.  Default workload is
configs[4] (c5): OPT-30B shapes, int4-g64 weights, b = 64 per GPU, prompt 512,
gen 32 (31 decode steps fit; more are allowed, positions keep growing).
Multi-GPU: one process per GPU (torchrun), batch-sharded, no collective on the
hot path; timing = max over ranks (device events), barrier on both sides.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import pipo_synth as synth  # noqa: E402

CONFIGS = {
    "c1": dict(shape=synth.OPTShape(768, 1, 12, 3072), b=4, P=32, G=8, weight_tier=1, kv_tier=0,
               desc="configs[0]: one OPT-125M-shaped decoder layer, int4 g64, b=4, P=32, gen 8"),
    "c2": dict(shape=synth.OPT_1_3B, b=16, P=256, G=32, weight_tier=1, kv_tier=0,
               desc="configs[1]: OPT-1.3B, weights in pinned host memory, b=16, P=256, gen 32"),
    "c3": dict(shape=synth.OPT_6_7B, b=32, P=512, G=32, weight_tier=1, kv_tier=1,
               desc="configs[2]: OPT-6.7B streamed weights + host-resident KV, b=32, P=512, gen 32"),
    "c4": dict(shape=synth.OPT_13B, b=64, P=512, G=32, weight_tier=2, kv_tier=0,
               desc="configs[3]: OPT-13B streamed weights from disk -> pinned host ring, b=64, P=512, gen 32"),
    "c5": dict(shape=synth.OPT_30B, b=64, P=512, G=32, weight_tier=1, kv_tier=0,
               desc="configs[4]: OPT-30B streamed weights, b=64/GPU, P=512, gen 32 (batch-sharded)"),
    # NEXT-4: the paper's LLaMA3.1 family (§4.1)
    "c6": dict(shape=synth.LLAMA31_8B, b=64, P=512, G=32, weight_tier=1, kv_tier=0,
               desc="NEXT-4: LLaMA3.1-8B streamed int4 weights (GQA 32/8, SwiGLU 14336, RoPE llama3), b=64, P=512, gen 32"),
    "c8": dict(shape=synth.LLAMA32_1B, b=1, P=512, G=32, weight_tier=1, kv_tier=0,
               desc="NEXT-4: LLaMA3.2-1B streamed int4 weights, b=1, P=512, gen 32 (the paper's offloading-overhead "
                    "table PAPER.md:727-742)"),
    "c7": dict(shape=synth.LLAMA31_8B, b=1, P=512, G=32, weight_tier=1, kv_tier=0,
               desc="NEXT-4: LLaMA3.1-8B streamed int4 weights, b=1, context 512, gen 32 (the paper's latency "
                    "table PAPER.md:697-713: TTFT + per-token decode latency)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="pipo", choices=["pipo", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--wfmt", default="int4", choices=["int4", "fp16"])
    ap.add_argument("--kv-fmt", default="fp16", choices=["fp16", "int4"],
                    help="KV cache storage (int4 = NEXT-2: PAPER.md:96 INT4 KV cache)")
    ap.add_argument("--ring", type=int, default=2)
    ap.add_argument("--weight-tier", default=None, choices=["device", "host", "disk"],
                    help="override the config's weight tier (device = no streaming: isolates H2D interference)")
    ap.add_argument("--chunk-mb", type=float, default=0)
    ap.add_argument("--prompt", type=int, default=0, help="override the config's prompt length P")
    ap.add_argument("--kv-tier", default=None, choices=["device", "host"], help="override the config's KV tier")
    ap.add_argument("--batch", type=int, default=0, help="override the config's per-GPU batch b")
    ap.add_argument("--shard-stream", action="store_true",
                    help="NEXT-1: each rank streams 1/N of every layer over its host link and all-gathers the "
                         "rest over NVLink (NCCL); compute stays batch-sharded (host weight tier only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cupti", action="store_true", help="skip the torch.profiler kernel-duration pass")
    ap.add_argument("--no-kprof", action="store_true",
                    help="no per-kernel timing events (no kernel roofline); A/B of the event overhead")
    ap.add_argument("--no-timeline", action="store_true",
                    help="no per-phase span events (busy fractions unavailable); A/B of the event overhead")
    ap.add_argument("--disk-dir", default="/tmp/pipo_disk")
    ap.add_argument("--profile", action="store_true",
                    help="cudaProfilerStart/Stop around the timed region (ncu --profile-from-start off)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[1]))
                mx = max(mx, float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def disk_probe(directory: str, threads: int = 4, chunk: int = 32 << 20) -> float:
    """Raw O_DIRECT read bandwidth (GB/s) of the layer blob files with `threads`
    concurrent readers and `chunk`-byte requests — the disk tier's roofline (App. A /
    Fig. 6 analogue)."""
    import mmap
    from concurrent.futures import ThreadPoolExecutor
    files = sorted(os.path.join(directory, f) for f in os.listdir(directory) if f.endswith(".pipo"))
    jobs = []
    for f in files:
        size = os.path.getsize(f)
        jobs += [(f, off, min(chunk, size - off)) for off in range(0, size, chunk)]
    bufs = [mmap.mmap(-1, chunk) for _ in range(threads)]
    flag = getattr(os, "O_DIRECT", 0)

    def work(t):
        buf, total = bufs[t], 0
        for f, off, n in jobs[t::threads]:
            fd = os.open(f, os.O_RDONLY | flag)
            try:
                n4 = (n + 4095) // 4096 * 4096
                total += os.preadv(fd, [memoryview(buf)[:n4]], off)
            finally:
                os.close(fd)
        return total

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        total = sum(ex.map(work, range(threads)))
    return total / (time.perf_counter() - t0) / 1e9


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------------------
class OracleSample:
    """The CPU oracle as it stands (oracle/opt.py), on a bounded sample of the
    workload: one decode step through ONE decoder layer at full batch b and
    L = P + G/2 cached positions, plus the LM head; a full step is extrapolated as
    n_layers * t_layer + t_head.  Weights are drawn once (setup, untimed)."""

    def __init__(self, cfg_name: str, wfmt: str):
        c = CONFIGS[cfg_name]
        self.s, self.b, P, G = c["shape"], c["b"], c["P"], c["G"]
        self.llama = isinstance(self.s, synth.LlamaShape)
        self.cores = len(os.sched_getaffinity(0))
        d = self.s.d_model
        if self.llama:
            from oracle import llama
            self.mod = llama
            self.lw = llama.layer_from_masters(synth.llama_layer_masters(self.s, 0), wfmt)
            spec = synth.llama_embed_tensor_specs(self.s)
            self.lnf = synth._draw_spec(synth.WEIGHT_SEED, 0, spec["lnf_g"]).astype(np.float64)
            self.head_w = synth._draw_spec(synth.WEIGHT_SEED, 0, spec["lm_head"]).astype(np.float64)
            self.inv = llama.rope_inv_freq(self.s.head_dim, self.s.rope_theta, self.s.rope_factor,
                                           self.s.rope_low_freq, self.s.rope_high_freq, self.s.rope_orig_max_pos)
            dkv = self.s.d_kv
        else:
            from oracle import opt
            self.mod = opt
            self.lw = opt.layer_from_masters(synth.layer_masters(self.s, 0), wfmt)
            emb = synth.embed_masters(self.s)
            self.lnf = (emb["lnf_g"].astype(np.float64), emb["lnf_b"].astype(np.float64))
            self.head_w = emb["tok"].astype(np.float64)
            dkv = d
        self.past = P + G // 2 - 1
        rng = np.random.default_rng(0)
        self.kc = rng.standard_normal((self.b, self.past + 1, dkv)) * 0.5
        self.vc = rng.standard_normal((self.b, self.past + 1, dkv)) * 0.5
        self.h = rng.standard_normal((self.b, 1, d))
        self.desc = (f"oracle/{'llama' if self.llama else 'opt'}.py fp64: 1 of {self.s.n_layers} decoder layers + "
                     f"LM head at b={self.b}, L={self.past + 1}, extrapolated x{self.s.n_layers} layers")

    def step(self) -> float:
        m = self.mod
        t0 = time.perf_counter()
        if self.llama:
            h2 = m.decoder_layer(self.h, self.lw, self.kc, self.vc, self.past, self.s.n_heads, self.s.n_kv_heads,
                                 self.inv)
            t1 = time.perf_counter()
            np.argmax(m.rms_norm(h2[:, 0], self.lnf) @ self.head_w.T, axis=-1)
        else:
            h2 = m.decoder_layer(self.h, self.lw, self.kc, self.vc, self.past, self.s.n_heads)
            t1 = time.perf_counter()
            m.greedy(m.layer_norm(h2[:, 0], *self.lnf) @ self.head_w.T)
        t2 = time.perf_counter()
        return (t1 - t0) * self.s.n_layers + (t2 - t1)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c = CONFIGS[args.config]
    sample = OracleSample(args.config, args.wfmt)
    t_all = []
    for i in range(args.warmup + args.steps):
        step = sample.step()
        if i >= args.warmup:
            t_all.append(step)
    ms = statistics.mean(t_all) * 1e3
    value = c["b"] / (ms / 1e3)
    line = {"impl": "reference", "metric": f"decode tokens/s, {c['desc']}", "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, "wfmt": args.wfmt},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": sample.cores, "kind": "oracle",
                             "sample": sample.desc},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def run_pipo(args):
    import torch
    import torch.distributed as dist

    from paper_2504_03664_b200 import pipo
    from paper_2504_03664_b200.shard import aggregate_throughput, max_over_ranks, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    if ndev == 0:
        raise SystemExit("bench.py needs a CUDA device (the library has no CPU path)")
    shared_gpu = world > ndev                  # smoke-testing N ranks on fewer GPUs
    local = local % ndev
    if world > 1:
        # plumbing only (barrier + max of device times): NCCL when every rank owns a GPU
        dist.init_process_group("gloo" if shared_gpu else "nccl")
    torch.cuda.set_device(local)
    c = CONFIGS[args.config]
    s, b, P, G = c["shape"], c["b"], c["P"], c["G"]
    if args.prompt:
        P = args.prompt   # context-length sweeps (the paper's latency table)
    if args.batch:
        b = args.batch
    steps_needed = args.warmup + args.steps * (2 if args.no_e2e else 3) + (0 if args.no_cupti else 2)
    max_seq = P + max(G, steps_needed + 1)
    if args.weight_tier:
        c = {**c, "weight_tier": ["device", "host", "disk"].index(args.weight_tier)}
    if args.kv_tier:
        c = {**c, "kv_tier": ["device", "host"].index(args.kv_tier)}
    disk_dir = f"{args.disk_dir}/rank{rank}" if c["weight_tier"] == 2 else None
    if disk_dir:
        os.makedirs(disk_dir, exist_ok=True)
    cfg = pipo.make_config(s, device=local, max_batch=b, max_seq=max_seq,
                           wfmt=pipo.PIPO_W_INT4_G64 if args.wfmt == "int4" else pipo.PIPO_W_FP16,
                           weight_tier=c["weight_tier"], kv_tier=c["kv_tier"], ring_layers=args.ring,
                           kv_fmt=pipo.PIPO_W_INT4_G64 if args.kv_fmt == "int4" else pipo.PIPO_W_FP16,
                           chunk_bytes=int(args.chunk_mb * (1 << 20)), disk_dir=disk_dir,
                           flags=(0 if args.no_timeline else pipo.PIPO_F_TIMELINE) |
                                 (0 if args.no_kprof else pipo.PIPO_F_KPROF))
    t_setup = time.perf_counter()
    pl = pipo.Pipeline(cfg)
    if args.shard_stream:
        uid = pipo.pipo_nccl_unique_id() if rank == 0 else bytes(128)
        if world > 1:
            t = torch.tensor(list(uid), dtype=torch.uint8, device="cpu" if shared_gpu else f"cuda:{local}")
            dist.broadcast(t, 0)
            uid = bytes(t.cpu().tolist())
        pipo.pipo_shard_stream_init(pl.ctx, rank, world, uid)
    pl.load_synthetic(pipo.PIPO_LAYER_EMBED, synth.WEIGHT_SEED)
    for j in range(s.n_layers):
        pl.load_synthetic(j, synth.WEIGHT_SEED)
    t_load = time.perf_counter() - t_setup
    link_probe = pipo.pipo_probe_h2d(pl.ctx, 256 << 20, 5)
    # App. A block-size sweep + Eq. (1) on this box (NEXT-3 planner, informational:
    # the configs force the streamed tier, reading Q19)
    sweep = [1 << 20, 4 << 20, 16 << 20, 32 << 20, 64 << 20, 128 << 20, 256 << 20]
    sweep_gbs = [pipo.pipo_probe_h2d(pl.ctx, n, 3) for n in sweep]
    # batch shard: rank r owns sequences [r*b, (r+1)*b) of the global prompt batch
    lo, hi = shard_range(b * world, world, rank)
    prompt = synth.prompts(b * world, P, s.vocab)[lo:hi]
    # TTFT: the first prefill of a fresh process also pays CUDA's lazy module loading
    # for every kernel it touches; the warm prefill (a second one, new batch) is the
    # serving number (the paper's latency table)
    t0 = time.perf_counter()
    nxt, _ = pl.prefill(prompt)
    t_prefill_cold = time.perf_counter() - t0
    pl.stats_reset()
    t0 = time.perf_counter()
    nxt, _ = pl.prefill(prompt)
    t_prefill = time.perf_counter() - t0
    for _ in range(args.warmup):
        nxt, _ = pl.decode_step(nxt)

    kpre = pipo.pipo_kernel_stats(pl.ctx)
    prefill_kernels = {n: {"ms": k["ms"], "tflops": k["flops"] / (k["ms"] / 1e3) / 1e12 if k["ms"] else 0.0,
                           "gbs": k["bytes"] / (k["ms"] / 1e3) / 1e9 if k["ms"] else 0.0}
                       for n, k in kpre.items() if n.endswith("prefill") and k["units"]}
    comp = torch.cuda.ExternalStream(pipo.pipo_stream(pl.ctx, 0), device=local)
    tok_dev = torch.from_numpy(nxt.astype(np.int32)).cuda(local)

    def barrier():
        torch.cuda.synchronize(local)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(local)

    # ---- value: inputs resident in HBM (device token ids, no host round trip) ----
    pl.stats_reset()
    barrier()
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if args.profile:
            torch.cuda.cudart().cudaProfilerStart()
        e0.record(comp)
        for _ in range(args.steps):
            pipo.decode_step_dev(pl.ctx, tok_dev.data_ptr(), tok_dev.data_ptr())
        e1.record(comp)
        torch.cuda.synchronize(local)
        if args.profile:
            torch.cuda.cudart().cudaProfilerStop()
    barrier()
    t_dev = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    st = pl.stats()
    kst = pipo.pipo_kernel_stats(pl.ctx)
    clocks = clk.summary()

    # ---- e2e: the public C-ABI call with HOST buffers, H2D ids + D2H ids every step ----
    e2e = None
    if not args.no_e2e:
        nxt = tok_dev.cpu().numpy()
        barrier()
        e0.record(comp)
        for _ in range(args.steps):
            nxt, _ = pl.decode_step(nxt)
        e1.record(comp)
        torch.cuda.synchronize(local)
        barrier()
        t_e2e = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        per_step_h2d = st["h2d_bytes"] / max(1, st["decode_steps"]) + b * 4
        e2e = {"value": aggregate_throughput(b, world, args.steps, t_e2e), "unit": "tokens/s",
               "h2d_bytes_per_step": int(per_step_h2d), "d2h_bytes_per_step": int(b * 4),
               "note": "decode_step(host tokens) -> host next ids; h2d counts the streamed weights too"}

    # Uninstrumented pass (same K steps, no timeline / per-kernel events): CUDA timing
    # events on the compute stream wait behind the copy engine (~25 us each, DESIGN.md
    # §12), which costs the small configs a few % of throughput; reported alongside.
    uninstr = None
    if rank == 0 or world > 1:
        pipo.pipo_set_flags(pl.ctx, 0)
        barrier()
        e0.record(comp)
        for _ in range(args.steps):
            pipo.decode_step_dev(pl.ctx, tok_dev.data_ptr(), tok_dev.data_ptr())
        e1.record(comp)
        torch.cuda.synchronize(local)
        barrier()
        t_un = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        pipo.pipo_set_flags(pl.ctx, pipo.PIPO_F_TIMELINE | pipo.PIPO_F_KPROF)
        un_ms = t_un / args.steps * 1e3
        uninstr = {"value": aggregate_throughput(b, world, args.steps, t_un), "ms_per_step": un_ms,
                   "link_frac": None,
                   "note": ("same K steps with PIPO_F_TIMELINE / PIPO_F_KPROF off (run after the timed and e2e "
                            "passes, i.e. at later KV positions: host-KV configs move more bytes)")}

    # CUPTI (torch.profiler) view of 2 extra untimed steps: true per-kernel GPU durations
    # with the copy stream running (context for the event-bracketed roofline above)
    cupti = None
    if not args.no_cupti and rank == 0:
        cupti = cupti_kernel_times(pl, tok_dev, 2, args.steps, kst)

    value = aggregate_throughput(b, world, args.steps, t_dev)
    ms = t_dev / args.steps * 1e3
    peaks = measured_peaks()
    layer_bytes = st["h2d_bytes"] / max(1, st["decode_steps"])
    link_floor_s = layer_bytes / (link_probe * 1e9)
    if uninstr and uninstr["ms_per_step"] > 0 and layer_bytes > 0:
        uninstr["link_frac"] = link_floor_s / (uninstr["ms_per_step"] / 1e3)
    kernels = {}
    for name, k in kst.items():
        if k["units"] and k["ms"] > 0:
            kernels[name] = {"units": k["units"], "ms_per_step": k["ms"] / args.steps,
                             "share_of_step": k["ms"] / args.steps / ms,
                             "gbs": k["bytes"] / (k["ms"] / 1e3) / 1e9, "tflops": k["flops"] / (k["ms"] / 1e3) / 1e12}
    dom = max(kernels, key=lambda n: kernels[n]["ms_per_step"]) if kernels else None
    roofline = None
    if dom:
        kd = kst[dom]
        per_unit_bytes = kd["bytes"] / kd["units"]
        per_unit_s = kd["ms"] / kd["units"] / 1e3
        hbm = peaks.get("hbm_gbs") or 6650.0
        tc = peaks.get("bf16_tflops_sustained") or 1400.0
        ach = per_unit_bytes / per_unit_s / 1e9
        roofline = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": ach / hbm, "traffic": ncu_traffic(dom, args),
                    "bytes_per_unit": per_unit_bytes, "us_per_unit": per_unit_s * 1e6,
                    "tflops": kd["flops"] / kd["units"] / per_unit_s / 1e12,
                    "tflops_frac_of_fp16_peak": kd["flops"] / kd["units"] / per_unit_s / 1e12 / tc,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy), bf16_tflops_sustained (fp16 same rate)",
                    "note": ("host/disk tier: CUDA timing events on the compute stream wait ~25 us behind the copy "
                             "engine's in-flight H2D command (DESIGN.md §12), so the event bracket over-counts; "
                             "roofline_cupti has the kernel-only time") if c["weight_tier"] != 0 else None}
    line = None
    if rank == 0:
        line = {
            "metric": "decode tokens/s, OPT-30B streamed weights (int4-g64), b=64/GPU, P=512" if args.config == "c5"
            else f"decode tokens/s, {c['desc']}",
            "decode_latency_ms": ms,
            "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16", "weights": args.wfmt + ("-g64" if args.wfmt == "int4" else ""),
            "data": "synthetic (seeded counter-based OPT weights + prompts, pipo_synth)",
            "config": {"workload": f"{args.config}: {c['desc']}", "global_batch": b * world, "seq_len": P,
                       "gen": G, "n_layers": s.n_layers, "d_model": s.d_model,
                       "parallelism": (f"batch-shard x{world} + sharded streaming (1/{world} of each layer over "
                                       f"PCIe, NCCL all-gather over NVLink)") if args.shard_stream
                       else f"batch-shard x{world} (no hot-path collective)",
                       "weight_tier": ["device", "host", "disk"][c["weight_tier"]],
                       "kv_tier": ["device", "host"][c["kv_tier"]], "kv_fmt": args.kv_fmt, "ring_layers": args.ring,
                       "l2": "inputs larger than L2 (every step streams all layer weights through HBM)"},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": int(st["kernel_launches"]),
            "roofline": roofline,
            "kernels": kernels,
            "roofline_cupti": cupti,
            "uninstrumented": uninstr,
            "link_roofline": {"bound": "host-link", "bytes_per_step": int(layer_bytes),
                              "probe_gbs": link_probe, "achieved_gbs": layer_bytes / (ms / 1e3) / 1e9,
                              "frac": link_floor_s / (ms / 1e3), "copy_engine_gbs": st["h2d_gbs"]},
            "busy": {"union": st["union_busy"], "copy": st["copy_busy"], "kernel": st["kernel_busy"]},
            "prefill_kernels": prefill_kernels,
            "setup": {"load_s": t_load, "prefill_s": t_prefill, "prefill_cold_s": t_prefill_cold,
                      "hbm_bytes": st["hbm_bytes"],
                      "pinned_host_bytes": st["pinned_host_bytes"]},
            "peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "bf16_tflops": peaks.get("bf16_tflops")},
        }
    pl.close()
    if rank == 0 and disk_dir:
        dgbs = disk_probe(disk_dir, threads=4)
        line["disk_roofline"] = {"bound": "disk (O_DIRECT, 4 readers, 32 MiB)", "probe_gbs": dgbs,
                                 "achieved_gbs": layer_bytes / (ms / 1e3) / 1e9,
                                 "frac": layer_bytes / (dgbs * 1e9) / (ms / 1e3)}
    if rank == 0:
        try:
            mem_cpu = int(open("/proc/meminfo").read().split("MemTotal:")[1].split()[0]) * 1024
        except (OSError, IndexError, ValueError):
            mem_cpu = 0
        b_ssd = (line.get("disk_roofline") or {}).get("probe_gbs")
        llama = isinstance(s, synth.LlamaShape)
        spec = pipo.mem_spec(l=s.n_layers, d=s.d_model, V=s.vocab, h=s.n_heads,
                             h_kv=s.n_kv_heads if llama else s.n_heads, d_h=s.ffn_dim,
                             mlp_mats=3 if llama else 2, p_weight=17 / 32 if args.wfmt == "int4" else 2.0, p_act=2.0)
        try:
            plan = pipo.pipo_choose_plan(spec, b, P + G, m_gpu=torch.cuda.get_device_properties(local).total_memory,
                                         m_cpu=mem_cpu or 1, b_gpu=link_probe * 1e9,
                                         b_ssd=(b_ssd or link_probe / 10) * 1e9,
                                         sizes=sweep, h2d_bps=[g * 1e9 for g in sweep_gbs])
            plan["weight_tier"] = ["device", "host", "disk"][plan["weight_tier"]]
            plan["b_ssd"] = "probed" if b_ssd else "not probed (assumed B_GPU/10)"
            plan["h2d_sweep_gbs"] = dict(zip([f"{n >> 20}MiB" for n in sweep], sweep_gbs))
            line["plan_eq1"] = plan
        except pipo.PipoError as e:
            line["plan_eq1"] = {"error": str(e)}
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        sample = OracleSample(args.config, args.wfmt)
        t = min(sample.step() for _ in range(2))
        line["cpu_baseline"] = {"value": b / t, "unit": "tokens/s", "cores": sample.cores, "kind": "oracle",
                                "sample": sample.desc + "; best of 2"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


_CLASS_KERNELS = {"linear_decode": ("gemm_tm_kernel", "gemm_ws_kernel", "gemv_int4_kernel", "ws_reduce",
                                     "gemm_tc_kernel"),
                  "attn_decode": ("attn_decode", "attn_merge")}


def cupti_kernel_times(pl, tok_dev, steps, timed_steps, kst):
    """Kernel-only GPU time per unit of each class from a CUPTI trace of `steps` extra
    decode steps (all of a class's kernels summed, e.g. the GEMM and its stream-K reduce;
    a PDL-launched reduce's span includes its wait, so this is an upper bound).  Units and
    algorithmic bytes per unit come from the event-timed region (`timed_steps` steps)."""
    import torch
    from paper_2504_03664_b200 import pipo
    try:
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            for _ in range(steps):
                pipo.decode_step_dev(pl.ctx, tok_dev.data_ptr(), tok_dev.data_ptr())
            torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001  (profiler unavailable: report, do not fail the bench)
        return {"error": str(e)[:200]}
    tot = {c: 0.0 for c in _CLASS_KERNELS}
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA:
            continue
        for c, names in _CLASS_KERNELS.items():
            if any(n in e.name for n in names):
                tot[c] += (e.time_range.end - e.time_range.start) * 1e-6
    out = {"source": f"torch.profiler CUDA activity (CUPTI), {steps} untimed steps after the timed region"}
    for c, t in tot.items():
        k = kst.get(c)
        if not k or not k["units"] or t <= 0:
            continue
        units_per_step = k["units"] / timed_steps
        us = t / steps / units_per_step * 1e6
        out[c] = {"us_per_unit": us, "gbs": k["bytes"] / k["units"] / (us * 1e-6) / 1e9}
    return out


def ncu_traffic(cls, args):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
    class's kernel from the committed `ncu --set full` capture (profiles/ncu_traffic.json,
    written by hand from tools/ncu_summary.py output), or None if that capture was not
    taken on this workload."""
    try:
        t = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")))
    except (OSError, ValueError):
        return None
    for ent in t.get("entries", [t]):   # one entry per captured workload
        want = ent.get("applies_to", {})
        if (want.get("config"), want.get("wfmt"), want.get("kv_fmt")) != (args.config, args.wfmt, args.kv_fmt):
            continue
        e = ent.get(cls)
        return None if e is None else e["traffic_bytes_per_unit"]
    return None


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_pipo(args)


if __name__ == "__main__":
    sys.exit(main())
