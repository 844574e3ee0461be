"""bench.py — decode tokens/s of the streamed-weight PIPO pipeline (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--wfmt int4|fp16]
    python bench.py --impl reference ...     # the CPU oracle arm (reads oracle/)

A "step" is one decode_step: all n_layers decoder layers (weights streamed from
pinned host memory over PCIe, chunk by chunk, consumed as they land) plus the LM
head and greedy argmax, for a batch of b sequences per GPU.  Default workload is
configs[4] (c5): OPT-30B shapes, int4-g64 weights, b = 64 per GPU, prompt 512,
gen 32 (31 decode steps fit; more are allowed, positions keep growing).

Multi-GPU: one process per GPU, batch-sharded, no collective on the hot path
(PAPER.md:809-812); timing = max over ranks (device events), barrier on both sides.
`--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N processes (127.0.0.1 rendezvous); it refuses to run
N ranks on fewer GPUs unless --allow-shared-gpu (a launcher test: ranks share GPU 0,
gloo plumbing).  At N > 1 the line also carries the all-N concurrent H2D probe and,
for the host tier, the NEXT-1 sharded-streaming variant timed in the same run
(`variants.shard_stream`).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# torchrun pins OMP_NUM_THREADS=1 per rank; rank 0 runs the CPU oracle (cpu_baseline /
# the reference arm) on all host cores, so it gets them back before numpy loads BLAS
if os.environ.get("RANK", "0") == "0" and os.environ.get("TORCHELASTIC_RUN_ID") and \
        os.environ.get("OMP_NUM_THREADS") == "1":
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[_v] = str(len(os.sched_getaffinity(0)))

import numpy as np  # noqa: E402

import pipo_synth as synth  # noqa: E402

CONFIGS = {
    "c1": dict(shape=synth.OPTShape(768, 1, 12, 3072), b=4, P=32, G=8, weight_tier=1, kv_tier=0,
               metric="one OPT-125M-shaped decoder layer, b=4, P=32, gen 8 (configs[0])",
               desc="configs[0]: one OPT-125M-shaped decoder layer, int4 g64, b=4, P=32, gen 8"),
    "c2": dict(shape=synth.OPT_1_3B, b=16, P=256, G=32, weight_tier=1, kv_tier=0,
               metric="OPT-1.3B weights in pinned host memory, b=16, P=256, gen 32 (configs[1])",
               desc="configs[1]: OPT-1.3B, weights in pinned host memory, b=16, P=256, gen 32"),
    "c3": dict(shape=synth.OPT_6_7B, b=32, P=512, G=32, weight_tier=1, kv_tier=1,
               metric="OPT-6.7B streamed weights + host-resident KV cache, b=32, P=512, gen 32 (configs[2])",
               desc="configs[2]: OPT-6.7B streamed weights + host-resident KV, b=32, P=512, gen 32"),
    "c4": dict(shape=synth.OPT_13B, b=64, P=512, G=32, weight_tier=2, kv_tier=0,
               metric="OPT-13B streamed weights from disk -> pinned host ring, b=64, P=512, gen 32 (configs[3])",
               desc="configs[3]: OPT-13B streamed weights from disk -> pinned host ring, b=64, P=512, gen 32"),
    "c5": dict(shape=synth.OPT_30B, b=64, P=512, G=32, weight_tier=1, kv_tier=0,
               metric="OPT-30B streamed weights, b=64/GPU, P=512, gen 32 (configs[4])",
               desc="configs[4]: OPT-30B streamed weights, b=64/GPU, P=512, gen 32 (batch-sharded)"),
    # NEXT-4: the paper's LLaMA3.1 family (§4.1)
    "c6": dict(shape=synth.LLAMA31_8B, b=64, P=512, G=32, weight_tier=1, kv_tier=0,
               metric="LLaMA3.1-8B streamed weights, b=64, P=512, gen 32 (NEXT-4)",
               desc="NEXT-4: LLaMA3.1-8B streamed int4 weights (GQA 32/8, SwiGLU 14336, RoPE llama3), b=64, P=512, gen 32"),
    "c8": dict(shape=synth.LLAMA32_1B, b=1, P=512, G=32, weight_tier=1, kv_tier=0,
               metric="LLaMA3.2-1B streamed weights, b=1, P=512, gen 32 (NEXT-4)",
               desc="NEXT-4: LLaMA3.2-1B streamed int4 weights, b=1, P=512, gen 32 (the paper's offloading-overhead "
                    "table PAPER.md:727-742)"),
    "c7": dict(shape=synth.LLAMA31_8B, b=1, P=512, G=32, weight_tier=1, kv_tier=0,
               metric="LLaMA3.1-8B streamed weights, b=1, context 512, gen 32 (NEXT-4)",
               desc="NEXT-4: LLaMA3.1-8B streamed int4 weights, b=1, context 512, gen 32 (the paper's latency "
                    "table PAPER.md:697-713: TTFT + per-token decode latency)"),
}
TIERS = ["device", "host", "disk"]


def parse(argv=None):
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
    ap.add_argument("--weight-tier", default=None, choices=TIERS,
                    help="override the config's weight tier (device = no streaming: isolates H2D interference)")
    ap.add_argument("--chunk-mb", type=float, default=0)
    ap.add_argument("--prompt", type=int, default=0, help="override the config's prompt length P")
    ap.add_argument("--kv-tier", default=None, choices=["device", "host"], help="override the config's KV tier")
    ap.add_argument("--batch", type=int, default=0, help="override the config's per-GPU batch b")
    ap.add_argument("--shard-stream", action="store_true",
                    help="NEXT-1 as the primary mode: each rank streams 1/N of every layer over its host link and "
                         "all-gathers the rest over NVLink (NCCL); compute stays batch-sharded (host tier only)")
    ap.add_argument("--shard-transport", default="p2p", choices=["p2p", "nccl"],
                    help="sharded streaming's gather: peer copies out of the peers' HBM rings through CUDA IPC "
                         "(p2p, the library's own transport) or an NCCL all-gather")
    ap.add_argument("--no-variants", action="store_true", help="N > 1: skip the sharded-streaming variant pass")
    ap.add_argument("--allow-shared-gpu", action="store_true",
                    help="let N ranks share fewer GPUs (launcher test only; gloo plumbing)")
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
    return ap.parse_args(argv)


def metric_name(args) -> str:
    """The SAME string in both arms (the driver pairs the lines by it)."""
    c = CONFIGS[args.config]
    fmt = "int4-g64" if args.wfmt == "int4" else "fp16"
    kv = ", int4 KV" if args.kv_fmt == "int4" else ""
    return f"decode tokens/s, {c['metric']}, {fmt} weights{kv}"


def workload(args):
    c = dict(CONFIGS[args.config])
    if args.prompt:
        c["P"] = args.prompt   # context-length sweeps (the paper's latency table)
    if args.batch:
        c["b"] = args.batch
    if args.weight_tier:
        c["weight_tier"] = TIERS.index(args.weight_tier)
    if args.kv_tier:
        c["kv_tier"] = ["device", "host"].index(args.kv_tier)
    return c


def workload_config(args, world: int) -> dict:
    """`config` of the JSON line: the workload only (identical in both arms)."""
    c = workload(args)
    s = c["shape"]
    return {"workload": f"{args.config}: {c['desc']}", "model": type(s).__name__, "global_batch": c["b"] * world,
            "seq_len": c["P"], "gen": c["G"], "n_layers": s.n_layers, "d_model": s.d_model,
            "wfmt": args.wfmt, "kv_fmt": args.kv_fmt,
            "weight_tier": TIERS[c["weight_tier"]], "kv_tier": ["device", "host"][c["kv_tier"]],
            "parallelism": (f"batch-shard x{world} + sharded streaming (1/{world} of each layer over PCIe, the rest "
                            f"gathered over NVLink, {args.shard_transport})") if args.shard_stream
            else f"batch-shard x{world} (no hot-path collective)",
            "l2": "inputs larger than L2 (every step streams all layer weights through HBM)"}


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


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def host_info() -> dict:
    info = {"cores": len(os.sched_getaffinity(0))}
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu"] = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        info["numa_nodes"] = len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")])
    except OSError:
        pass
    return info


# ---------------------------------------------------------------------------
def _decode_step_counts(s, b: int, L: int) -> tuple[float, float]:
    """Algorithmic (flops, fp64 bytes) of ONE oracle decode step of the whole model at
    L attended positions: every linear weight, the KV cache and the LM head are read
    once in float64 (the oracle holds them as float64); 2 flops per multiply-add."""
    llama = isinstance(s, synth.LlamaShape)
    d, l, V = s.d_model, s.n_layers, s.vocab
    dkv = s.d_kv if llama else d
    lin = d * (d + 2 * dkv) + d * d + (3 if llama else 2) * d * s.ffn_dim
    flops = l * (2.0 * b * lin + 4.0 * b * d * L) + 2.0 * b * V * d
    byts = l * (8.0 * lin + 2 * 8.0 * b * L * dkv) + 8.0 * V * d
    return flops, byts


class OracleRun:
    """The CPU oracle as it stands (oracle/opt.py, oracle/llama.py: float64, one library
    matmul per product), on the host cores.

    full=True (c1, c2: SURVEY.md §8(d) "timed fully on c1 and on c2"): the real
    workload — the whole model, prefill of the b x P prompt in setup (timed as TTFT),
    then every step() is one real decode step of the greedy generation (positions keep
    growing past P + G if more steps are asked for).
    full=False (c3..c8): a bounded sample — one decode step through ONE decoder layer at
    the full batch and L = P + G/2 cached positions, plus the LM head; the whole step is
    extrapolated as n_layers * t_layer + t_head (labelled "extrapolated")."""

    def __init__(self, cfg: dict, wfmt: str, full: bool, max_steps: int = 64):
        self.s, self.b, self.P, self.G = cfg["shape"], cfg["b"], cfg["P"], cfg["G"]
        self.full = full
        self.llama = isinstance(self.s, synth.LlamaShape)
        self.cores = len(os.sched_getaffinity(0))
        s, d = self.s, self.s.d_model
        t0 = time.perf_counter()
        if full:
            prompt = synth.prompts(self.b, self.P, s.vocab)
            s_max = self.P + max(self.G, max_steps + 1)
            if self.llama:
                from oracle import llama
                self.model = llama.OracleLlama.from_masters(
                    s, synth.llama_embed_masters(s), [synth.llama_layer_masters(s, j) for j in range(s.n_layers)],
                    wfmt, s_max)
                self._greedy = lambda lg: np.argmax(lg, axis=-1).astype(np.int32)
            else:
                from oracle import opt
                self.model = opt.OracleOPT.from_masters(
                    s.n_heads, synth.embed_masters(s), [synth.layer_masters(s, j) for j in range(s.n_layers)],
                    wfmt, s_max)
                self._greedy = opt.greedy
            self.setup_s = time.perf_counter() - t0
            t1 = time.perf_counter()
            self.ids = self._greedy(self.model.prefill(prompt))
            self.ttft_s = time.perf_counter() - t1
            self.desc = (f"oracle/{'llama' if self.llama else 'opt'}.py float64, the whole {s.n_layers}-layer model: "
                         f"prefill b={self.b} x P={self.P} in setup, each step one real greedy decode step")
            return
        d = s.d_model
        if self.llama:
            from oracle import llama
            self.mod = llama
            self.lw = llama.layer_from_masters(synth.llama_layer_masters(s, 0), wfmt)
            spec = synth.llama_embed_tensor_specs(s)
            self.lnf = synth._draw_spec(synth.WEIGHT_SEED, 0, spec["lnf_g"]).astype(np.float64)
            self.head_w = synth._draw_spec(synth.WEIGHT_SEED, 0, spec["lm_head"]).astype(np.float64)
            self.inv = llama.rope_inv_freq(s.head_dim, s.rope_theta, s.rope_factor, s.rope_low_freq,
                                           s.rope_high_freq, s.rope_orig_max_pos)
            dkv = s.d_kv
        else:
            from oracle import opt
            self.mod = opt
            self.lw = opt.layer_from_masters(synth.layer_masters(s, 0), wfmt)
            emb = synth.embed_masters(s)
            self.lnf = (emb["lnf_g"].astype(np.float64), emb["lnf_b"].astype(np.float64))
            self.head_w = emb["tok"].astype(np.float64)
            dkv = d
        self.past = self.P + self.G // 2 - 1
        rng = np.random.default_rng(0)
        self.kc = rng.standard_normal((self.b, self.past + 1, dkv)) * 0.5
        self.vc = rng.standard_normal((self.b, self.past + 1, dkv)) * 0.5
        self.h = rng.standard_normal((self.b, 1, d))
        self.setup_s = time.perf_counter() - t0
        self.ttft_s = None
        self.desc = (f"oracle/{'llama' if self.llama else 'opt'}.py float64: 1 of {s.n_layers} decoder layers + "
                     f"LM head at b={self.b}, L={self.past + 1}; step extrapolated x{s.n_layers} layers")

    def step(self) -> tuple[float, float]:
        """One step: returns (seconds actually spent, seconds of the whole model step
        — equal for full runs, extrapolated for samples)."""
        if self.full:
            t0 = time.perf_counter()
            self.ids = self._greedy(self.model.decode(self.ids))
            t = time.perf_counter() - t0
            return t, t
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
        return t2 - t0, (t1 - t0) * self.s.n_layers + (t2 - t1)

    def counts(self, L: int) -> tuple[float, float]:
        return _decode_step_counts(self.s, self.b, L)

    def baseline(self, n_steps: int) -> dict:
        """cpu_baseline object: tokens/s of the whole-model step, achieved GFLOP/s and
        GB/s (algorithmic float64 bytes) of what was executed, cores, sample."""
        spent, full = [], []
        L0 = self.P + 1 if self.full else self.past + 1
        for _ in range(n_steps):
            a, f = self.step()
            spent.append(a)
            full.append(f)
        t_full = statistics.median(full)
        L = L0 + (n_steps // 2 if self.full else 0)
        fl, by = self.counts(L)
        return {"value": self.b / t_full, "unit": "tokens/s", "cores": self.cores, "kind": "oracle",
                "extrapolated": not self.full, "sample": self.desc + f"; median of {n_steps} steps",
                "step_s": t_full, "sample_s": statistics.median(spent),
                "gflops": fl / t_full / 1e9, "gbs_fp64": by / t_full / 1e9,
                "ttft_s": self.ttft_s, "host": host_info()}


def oracle_full_for(config: str) -> bool:
    return config in ("c1", "c2")


def run_reference(args):
    """The reference arm: the CPU oracle (this tier's rule), rank 0 only."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    world = max(args.gpus, int(os.environ.get("WORLD_SIZE", "1")))
    c = workload(args)
    run = OracleRun(c, args.wfmt, oracle_full_for(args.config), max_steps=args.warmup + args.steps)
    for _ in range(args.warmup):
        run.step()
    spent, full = [], []
    for _ in range(args.steps):
        a, f = run.step()
        spent.append(a)
        full.append(f)
    t_full = statistics.mean(full)
    value = c["b"] / t_full
    L = (run.P + 1 + args.warmup + args.steps // 2) if run.full else run.past + 1
    fl, by = run.counts(L)
    line = {"impl": "reference", "metric": metric_name(args), "value": value, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            # the time of what actually ran per step (a one-layer sample for c3..c8), so
            # steps x ms_per_step is this process's own timed wall time
            "ms_per_step": statistics.mean(spent) * 1e3,
            "extrapolated": not run.full,
            "extrapolated_ms_per_step": None if run.full else t_full * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded pipo_synth weights + prompts)", "config": workload_config(args, world),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": run.cores, "kind": "oracle",
                             "extrapolated": not run.full, "sample": run.desc,
                             "gflops": fl / t_full / 1e9, "gbs_fp64": by / t_full / 1e9,
                             "ttft_s": run.ttft_s, "setup_s": run.setup_s, "host": host_info()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
_CLASS_KERNELS = {"linear_decode": ("gemm_tm_kernel", "gemm_ws_kernel", "gemv_int4_kernel", "ws_reduce",
                                     "gemm_tc_kernel", "gemm_dec"),
                  "attn_decode": ("attn_decode", "attn_merge"),
                  "lm_head": ("gemm_kernel", "lm_head")}


def exclusive_class_times(events, classes):
    """Kernel time per class from (stream, start_us, end_us, name) device events: each
    kernel counts only the part of [start, end] after every earlier kernel of its stream
    has ended.  Kernels are launched with programmatic dependent launch, so a kernel
    "starts" while its predecessor drains (its CTAs wait in griddepcontrol.wait); raw
    durations would count that overlap twice (a GEMM + its overlapping stream-K reduce).
    Memcpy/memset events are skipped: the copy engines overlap the kernels by design.
    Returns ({class: seconds}, {class: set(kernel names)}, number of streams)."""
    by_stream = {}
    for sid, a, b, name in events:
        if name.startswith(("Memcpy", "Memset")):
            continue
        by_stream.setdefault(sid, []).append((a, b, name))
    tot = {c: 0.0 for c in classes}
    names = {}
    for evs in by_stream.values():
        run_end = None
        for a, b, name in sorted(evs):
            excl = max(0.0, b - (a if run_end is None else max(a, run_end)))
            run_end = b if run_end is None else max(run_end, b)
            for c, pats in classes.items():
                if any(n in name for n in pats):
                    tot[c] += excl * 1e-6
                    names.setdefault(c, set()).add(name.split("(")[0].split("<")[0])
                    break
    return tot, names, len(by_stream)


def cupti_kernel_times(pl, tok_dev, steps, timed_steps, kst, profile: bool):
    """Kernel-only GPU time per unit of each class from a CUPTI trace (torch.profiler)
    of `steps` extra decode steps run right after the timed region (each kernel's time
    exclusive of its stream predecessors, so PDL overlap is not counted twice).  Units and algorithmic bytes
    per unit come from the event-timed region (`timed_steps` steps).  Every rank runs
    the steps (the sharded variant has a collective); only `profile` ranks trace."""
    import torch
    from paper_2504_03664_b200 import pipo
    if not profile:
        for _ in range(steps):
            pipo.decode_step_dev(pl.ctx, tok_dev.data_ptr(), tok_dev.data_ptr())
        torch.cuda.synchronize()
        return None
    try:
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            for _ in range(steps):
                pipo.decode_step_dev(pl.ctx, tok_dev.data_ptr(), tok_dev.data_ptr())
            torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001  (profiler unavailable: report, do not fail the bench)
        return {"error": str(e)[:200]}
    evs = [(getattr(e, "device_resource_id", None) if getattr(e, "device_resource_id", None) is not None else e.thread,
            e.time_range.start, e.time_range.end, e.name)
           for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    tot, names, n_streams = exclusive_class_times(evs, _CLASS_KERNELS)
    out = {"source": f"torch.profiler CUDA activity (CUPTI), {steps} untimed, uninstrumented steps right after the timed region; "
                     "per kernel its exclusive time on its stream (after every earlier kernel of the stream ended)",
           "streams": n_streams}
    for c, t in tot.items():
        k = kst.get(c)
        if not k or not k["units"] or t <= 0:
            continue
        units_per_step = k["units"] / timed_steps
        us = t / steps / units_per_step * 1e6
        out[c] = {"us_per_unit": us, "ms_per_step": t / steps * 1e3, "units_per_step": units_per_step,
                  "bytes_per_unit": k["bytes"] / k["units"], "flops_per_unit": k["flops"] / k["units"],
                  "kernels": sorted(names.get(c, []))}
    return out


def roofline_of(cupti: dict | None, kernels: dict, kst: dict, steps: int, peaks: dict):
    """The `roofline` object for the dominant kernel class (largest kernel-only time per
    step): bound = the slower of HBM (algorithmic bytes / measured copy bandwidth) and
    tensor (flops / measured sustained bf16 = fp16 dense rate), achieved and frac against
    that bound, per unit timed by CUPTI (kernel-only; the event-bracketed time carries
    ~25 us of event latency per unit in the host tier)."""
    hbm = peaks.get("hbm_gbs") or 6650.0
    tc = peaks.get("bf16_tflops_sustained") or 1400.0
    src = "cupti"
    table = {c: v for c, v in (cupti or {}).items() if isinstance(v, dict) and "us_per_unit" in v}
    if not table:   # no CUPTI: fall back to the event-bracketed units
        src = "cuda_events"
        table = {c: {"us_per_unit": kst[c]["ms"] / kst[c]["units"] * 1e3,
                     "ms_per_step": kst[c]["ms"] / steps, "bytes_per_unit": kst[c]["bytes"] / kst[c]["units"],
                     "flops_per_unit": kst[c]["flops"] / kst[c]["units"]}
                 for c in kernels}
    if not table:
        return None
    dom = max(table, key=lambda c: table[c]["ms_per_step"])

    def frac_of(v):
        tt = v["us_per_unit"] * 1e-6
        th, tc_ = v["bytes_per_unit"] / (hbm * 1e9), v["flops_per_unit"] / (tc * 1e12)
        return {"bound": "tensor" if tc_ > th else "hbm", "frac": max(th, tc_) / tt, "us_per_unit": v["us_per_unit"],
                "ms_per_step": v["ms_per_step"]}
    by_class = {c: frac_of(v) for c, v in table.items()}
    u = table[dom]
    t = u["us_per_unit"] * 1e-6
    t_hbm = u["bytes_per_unit"] / (hbm * 1e9)
    t_tc = u["flops_per_unit"] / (tc * 1e12)
    tensor = t_tc > t_hbm
    ev = kernels.get(dom)
    return {"kernel": dom, "bound": "tensor" if tensor else "hbm",
            "achieved": (u["flops_per_unit"] / t / 1e12) if tensor else (u["bytes_per_unit"] / t / 1e9),
            "peak": tc if tensor else hbm, "unit": "TFLOP/s" if tensor else "GB/s",
            "frac": max(t_hbm, t_tc) / t, "traffic": None, "timing": src,
            "us_per_unit": u["us_per_unit"], "bytes_per_unit": u["bytes_per_unit"],
            "flops_per_unit": u["flops_per_unit"], "t_hbm_us": t_hbm * 1e6, "t_tensor_us": t_tc * 1e6,
            "frac_hbm": t_hbm / t, "frac_tensor": t_tc / t,
            "event_us_per_unit": (ev["ms_per_step"] * steps / ev["units"] * 1e3) if ev else None,
            "peak_source": "MEASURED_PEAKS.json: hbm_gbs (copy) / bf16_tflops_sustained (fp16 dense = bf16 rate)",
            "by_class": by_class}


def ncu_traffic(cls, args):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
    class's kernel from the committed `ncu --set full` capture (profiles/ncu_traffic.json,
    written from tools/ncu_summary.py output), or None if that capture was not taken
    on this workload."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    except (OSError, ValueError):
        return None
    for ent in t.get("entries", [t]):   # one entry per captured workload
        want = ent.get("applies_to", {})
        if (want.get("config"), want.get("wfmt"), want.get("kv_fmt")) != (args.config, args.wfmt, args.kv_fmt):
            continue
        e = ent.get(cls)
        return None if e is None else e["traffic_bytes_per_unit"]
    return None


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
    if args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    shared_gpu = world > ndev
    if shared_gpu and not args.allow_shared_gpu:
        raise SystemExit(f"{world} ranks need {world} GPUs, found {ndev} (--allow-shared-gpu for a launcher test)")
    local = local % ndev
    if world > 1:
        # plumbing only (barrier + max of device times): NCCL when every rank owns a GPU
        dist.init_process_group("gloo" if shared_gpu else "nccl")
    torch.cuda.set_device(local)
    # NUMA: this rank's host threads on its GPU's socket (the library binds the pinned
    # stores themselves, pipo_config.numa_node = GPU-local)
    node = pipo.pipo_gpu_numa_node(local)
    info = host_info()
    if node >= 0 and info.get("numa_nodes", 1) > 1:
        try:
            cpus = open(f"/sys/devices/system/node/node{node}/cpulist").read().strip()
            ids = set()
            for part in cpus.split(","):
                a, _, b_ = part.partition("-")
                ids.update(range(int(a), int(b_ or a) + 1))
            os.sched_setaffinity(0, ids)
        except (OSError, ValueError):
            pass
    c = workload(args)
    s, b, P, G = c["shape"], c["b"], c["P"], c["G"]
    steps_needed = args.warmup + args.steps * (2 if args.no_e2e else 3) + (0 if args.no_cupti else 3)
    max_seq = P + max(G, steps_needed + 1)
    disk_dir = f"{args.disk_dir}/rank{rank}" if c["weight_tier"] == 2 else None
    if disk_dir:
        os.makedirs(disk_dir, exist_ok=True)
    flags = (0 if args.no_timeline else pipo.PIPO_F_TIMELINE) | (0 if args.no_kprof else pipo.PIPO_F_KPROF)

    def gather_list(x):
        if world == 1:
            return [x]
        out = [None] * world
        dist.all_gather_object(out, x)
        return out

    def make_pipeline(shard: bool):
        cfg = pipo.make_config(s, device=local, max_batch=b, max_seq=max_seq,
                               wfmt=pipo.PIPO_W_INT4_G64 if args.wfmt == "int4" else pipo.PIPO_W_FP16,
                               weight_tier=c["weight_tier"], kv_tier=c["kv_tier"],
                               ring_layers=max(args.ring, 3) if shard else args.ring,
                               kv_fmt=pipo.PIPO_W_INT4_G64 if args.kv_fmt == "int4" else pipo.PIPO_W_FP16,
                               chunk_bytes=int(args.chunk_mb * (1 << 20)), disk_dir=disk_dir, flags=flags)
        t0 = time.perf_counter()
        pl = pipo.Pipeline(cfg)
        if shard and args.shard_transport == "p2p":
            h = pipo.pipo_shard_p2p_export(pl.ctx, rank, world)
            pipo.pipo_shard_p2p_init(pl.ctx, gather_list(h))
        elif shard:
            uid = pipo.pipo_nccl_unique_id() if rank == 0 else bytes(128)
            if world > 1:
                t = torch.tensor(list(uid), dtype=torch.uint8, device="cpu" if shared_gpu else f"cuda:{local}")
                dist.broadcast(t, 0)
                uid = bytes(t.cpu().tolist())
            pipo.pipo_shard_stream_init(pl.ctx, rank, world, uid)
        pl.load_synthetic(pipo.PIPO_LAYER_EMBED, synth.WEIGHT_SEED)
        for j in range(s.n_layers):
            pl.load_synthetic(j, synth.WEIGHT_SEED)
        return pl, time.perf_counter() - t0

    def barrier():
        torch.cuda.synchronize(local)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(local)

    pl, t_load = make_pipeline(args.shard_stream)
    link_probe = pipo.pipo_probe_h2d(pl.ctx, 256 << 20, 5)
    # all-N concurrent probe: every rank's link at once (shared host memory / PCIe
    # switches show up here, SURVEY.md §8(e) risks)
    barrier()
    conc = gather_list(pipo.pipo_probe_h2d(pl.ctx, 256 << 20, 5)) if world > 1 else None
    # App. A block-size sweep + Eq. (1) on this box (NEXT-3 planner)
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

    def timed_dev_steps(n):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(comp)
        for _ in range(n):
            pipo.decode_step_dev(pl.ctx, tok_dev.data_ptr(), tok_dev.data_ptr())
        e1.record(comp)
        torch.cuda.synchronize(local)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / 1e3)

    # ---- value: inputs resident in HBM (device token ids, no host round trip) ----
    pl.stats_reset()
    with ClockSampler(local) as clk:
        if args.profile:
            torch.cuda.cudart().cudaProfilerStart()
        t_dev = timed_dev_steps(args.steps)
        if args.profile:
            torch.cuda.cudart().cudaProfilerStop()
    st = pl.stats()
    kst = pipo.pipo_kernel_stats(pl.ctx)
    clocks = clk.summary()

    # ---- e2e: the public C-ABI call with HOST buffers, H2D ids + D2H ids every step ----
    e2e = None
    if not args.no_e2e:
        nxt = tok_dev.cpu().numpy()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(comp)
        for _ in range(args.steps):
            nxt, _ = pl.decode_step(nxt)
        e1.record(comp)
        torch.cuda.synchronize(local)
        barrier()
        t_e2e = max_over_ranks(e0.elapsed_time(e1) / 1e3)
        tok_dev.copy_(torch.from_numpy(nxt.astype(np.int32)))
        per_step_h2d = st["h2d_bytes"] / max(1, st["decode_steps"]) + b * 4
        e2e = {"value": aggregate_throughput(b, world, args.steps, t_e2e), "unit": "tokens/s",
               "h2d_bytes_per_step": int(per_step_h2d), "d2h_bytes_per_step": int(b * 4),
               "note": "decode_step(host tokens) -> host next ids; h2d counts the streamed weights too"}

    # Uninstrumented pass (same K steps, no timeline / per-kernel events): CUDA timing
    # events on the compute stream wait behind the copy engine (~25 us each, DESIGN.md
    # §12), which costs the small configs a few % of throughput; reported alongside.
    pipo.pipo_set_flags(pl.ctx, 0)
    t_un = timed_dev_steps(args.steps)
    pipo.pipo_set_flags(pl.ctx, flags)
    un_ms = t_un / args.steps * 1e3
    uninstr = {"value": aggregate_throughput(b, world, args.steps, t_un), "ms_per_step": un_ms, "link_frac": None,
               "note": ("same K steps with PIPO_F_TIMELINE / PIPO_F_KPROF off (run after the timed and e2e passes, "
                        "i.e. at later KV positions: host-KV configs move more bytes)")}

    # CUPTI (torch.profiler) view of 3 extra steps: true per-kernel GPU durations with the
    # copy stream running — the roofline's timing
    # (run uninstrumented: no timing events between the kernels, the production launch
    # sequence with its programmatic-dependent-launch overlaps)
    cupti = None
    if not args.no_cupti:
        pipo.pipo_set_flags(pl.ctx, 0)
        cupti = cupti_kernel_times(pl, tok_dev, 3, args.steps, kst, profile=(rank == 0))
        pipo.pipo_set_flags(pl.ctx, flags)

    value = aggregate_throughput(b, world, args.steps, t_dev)
    ms = t_dev / args.steps * 1e3
    peaks = measured_peaks()
    layer_bytes = st["h2d_bytes"] / max(1, st["decode_steps"])
    link_floor_s = layer_bytes / (link_probe * 1e9)
    if un_ms > 0 and layer_bytes > 0:
        uninstr["link_frac"] = link_floor_s / (un_ms / 1e3)
    kernels = {}
    for name, k in kst.items():
        if k["units"] and k["ms"] > 0:
            kernels[name] = {"units": k["units"], "ms_per_step": k["ms"] / args.steps,
                             "share_of_step": k["ms"] / args.steps / ms,
                             "gbs": k["bytes"] / (k["ms"] / 1e3) / 1e9, "tflops": k["flops"] / (k["ms"] / 1e3) / 1e12,
                             "timing": "cuda_events (include ~25 us event latency per unit in streamed tiers)"}
    roofline = roofline_of(cupti, kernels, kst, args.steps, peaks) if rank == 0 else None
    if roofline:
        roofline["traffic"] = ncu_traffic(roofline["kernel"], args)
    stats_all = gather_list({k: st[k] for k in ("union_busy", "copy_busy", "kernel_busy", "h2d_gbs", "numa_node",
                                                "numa_local_frac", "timeline_truncated")})
    line = None
    if rank == 0:
        line = {
            "metric": metric_name(args),
            "decode_latency_ms": ms,
            "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16", "weights": args.wfmt + ("-g64" if args.wfmt == "int4" else ""),
            "data": "synthetic (seeded counter-based OPT/LLaMA weights + prompts, pipo_synth)",
            "config": workload_config(args, world),
            "run": {"ring_layers": args.ring, "chunk_mb": args.chunk_mb, "shared_gpu": shared_gpu},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": int(st["kernel_launches"]),
            "roofline": roofline,
            "kernels": kernels,
            "roofline_cupti": cupti,
            "uninstrumented": uninstr,
            "link_roofline": {"bound": "host-link", "bytes_per_step": int(layer_bytes),
                              "probe_gbs": link_probe, "achieved_gbs": layer_bytes / (ms / 1e3) / 1e9,
                              "frac": link_floor_s / (ms / 1e3), "copy_engine_gbs": st["h2d_gbs"],
                              "concurrent_probe_gbs": conc,
                              "concurrent_frac": (min(conc) / link_probe) if conc else None},
            "busy": {"union": st["union_busy"], "copy": st["copy_busy"], "kernel": st["kernel_busy"],
                     "per_rank": stats_all if world > 1 else None},
            "numa": {"node": st["numa_node"], "local_frac": st["numa_local_frac"], "gpu_node": node,
                     "host_nodes": info.get("numa_nodes")},
            "prefill_kernels": prefill_kernels,
            "setup": {"load_s": t_load, "prefill_s": t_prefill, "prefill_cold_s": t_prefill_cold,
                      "hbm_bytes": st["hbm_bytes"],
                      "pinned_host_bytes": st["pinned_host_bytes"]},
            "peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "bf16_tflops": peaks.get("bf16_tflops"),
                      "bf16_tflops_sustained": peaks.get("bf16_tflops_sustained")},
        }
    pl.close()

    # ---- NEXT-1 variant at N > 1: sharded streaming timed in the same run ----
    if world > 1 and not args.no_variants and not args.shard_stream and c["weight_tier"] == 1 and \
            (args.shard_transport == "p2p" or not shared_gpu):   # NCCL refuses two ranks on one GPU
        try:
            pv, t_load_v = make_pipeline(True)
            nv, _ = pv.prefill(prompt)
            for _ in range(args.warmup):
                nv, _ = pv.decode_step(nv)
            pv.stats_reset()
            tok_v = torch.from_numpy(nv.astype(np.int32)).cuda(local)
            comp_v = torch.cuda.ExternalStream(pipo.pipo_stream(pv.ctx, 0), device=local)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(comp_v)
            for _ in range(args.steps):
                pipo.decode_step_dev(pv.ctx, tok_v.data_ptr(), tok_v.data_ptr())
            e1.record(comp_v)
            torch.cuda.synchronize(local)
            barrier()
            t_v = max_over_ranks(e0.elapsed_time(e1) / 1e3)
            sv = pv.stats()
            pv.close()
            if rank == 0:
                per_rank_link = sv["h2d_bytes"] / max(1, sv["decode_steps"])
                line["variants"] = {"shard_stream": {
                    "value": aggregate_throughput(b, world, args.steps, t_v), "ms_per_step": t_v / args.steps * 1e3,
                    "per_rank_link_bytes_per_step": int(per_rank_link),
                    "link_frac": per_rank_link / (link_probe * 1e9) / (t_v / args.steps),
                    "union_busy": sv["union_busy"], "load_s": t_load_v,
                    "transport": args.shard_transport,
                    "how": "each rank streams 1/N of every layer over its own PCIe link; the other ranges come from "
                           "the peers' HBM rings over NVLink on a gather stream (p2p: copy-engine pulls through CUDA "
                           "IPC ordered by flags in peer memory; nccl: all-gather), ring 3; compute batch-sharded as "
                           "the main line"}}
        except Exception as e:  # noqa: BLE001  (report the variant's failure, keep the main line)
            if rank == 0:
                line["variants"] = {"shard_stream": {"error": str(e)[:300]}}

    if rank == 0 and disk_dir:
        # the library's probe: the reader pool's read path (4 threads, O_DIRECT, the tier's
        # 32 MiB or --chunk-mb chunks) without the GPU handshake, over the same layer files
        chunk = int(args.chunk_mb * (1 << 20)) if args.chunk_mb else 32 << 20
        chunk = max(4096, chunk // 4096 * 4096)
        dgbs, _ = pipo.pipo_probe_disk(disk_dir, s.n_layers, 4, chunk)
        ach = layer_bytes / (ms / 1e3) / 1e9
        line["disk_roofline"] = {"bound": "disk", "probe_gbs": dgbs, "achieved_gbs": ach, "frac": ach / dgbs,
                                 "probe": "pipo_probe_disk: 4 reader threads, O_DIRECT, %d MiB chunks, all %d "
                                          "layer files once, no GPU handshake" % (chunk >> 20, s.n_layers)}
    if rank == 0:
        try:
            mem_cpu = int(open("/proc/meminfo").read().split("MemTotal:")[1].split()[0]) * 1024
        except (OSError, IndexError, ValueError):
            mem_cpu = 0
        llama = isinstance(s, synth.LlamaShape)
        spec = pipo.mem_spec(l=s.n_layers, d=s.d_model, V=s.vocab, h=s.n_heads,
                             h_kv=s.n_kv_heads if llama else s.n_heads, d_h=s.ffn_dim,
                             mlp_mats=3 if llama else 2, p_weight=17 / 32 if args.wfmt == "int4" else 2.0, p_act=2.0)
        try:
            plan = pipo.pipo_choose_plan(spec, b, P + G, m_gpu=torch.cuda.get_device_properties(local).total_memory,
                                         m_cpu=mem_cpu or 1, b_gpu=link_probe * 1e9, b_ssd=link_probe / 10 * 1e9,
                                         sizes=sweep, h2d_bps=[g * 1e9 for g in sweep_gbs])
            plan["weight_tier"] = TIERS[plan["weight_tier"]]
            plan["b_ssd"] = "not probed (assumed B_GPU/10)"
            plan["h2d_sweep_gbs"] = dict(zip([f"{n >> 20}MiB" for n in sweep], sweep_gbs))
            line["plan_eq1"] = plan
        except pipo.PipoError as e:
            line["plan_eq1"] = {"error": str(e)}
        if not args.no_cpu_baseline:
            # bounded sample (~10-30 s of host CPU work), rank 0 only, after the GPU passes
            run = OracleRun(c, args.wfmt, oracle_full_for(args.config), max_steps=8)
            n = 8 if run.full else max(2, min(8, int(15.0 / max(0.05, run.step()[0]))))
            line["cpu_baseline"] = run.baseline(n)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args) -> int:
    """`--gpus N` outside torchrun: re-run this script as N ranks under
    torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous)."""
    if args.impl == "pipo" and not args.allow_shared_gpu:
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            raise SystemExit(f"--gpus {args.gpus}: only {n} CUDA device(s) visible (no shared-GPU fallback; "
                             "--allow-shared-gpu for a launcher test)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_pipo(args)


if __name__ == "__main__":
    sys.exit(main())
