"""Probe a GPU box: host RAM, CPU, NUMA, topology, NVMe, H2D/D2H bandwidth (pinned)."""
import os, subprocess, json, time
out = {}
def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)
out["free"] = sh("free -g")
out["nproc"] = sh("nproc")
out["affinity"] = len(os.sched_getaffinity(0))
out["lscpu"] = sh("lscpu | head -30")
out["numactl"] = sh("numactl -H 2>&1 | head -20")
out["topo"] = sh("nvidia-smi topo -m")
out["smi"] = sh("nvidia-smi")
out["lsblk"] = sh("lsblk -o NAME,SIZE,TYPE,MOUNTPOINT,ROTA,MODEL 2>&1")
out["df"] = sh("df -h / /tmp /dev/shm 2>&1")
out["ulimit_l"] = sh("ulimit -l")
out["nvme"] = sh("ls /dev/nvme* 2>&1; cat /proc/mounts | head -40")
import torch
dev = torch.device("cuda:0")
res = {}
for mb in [1, 4, 16, 32, 64, 128, 256, 1024]:
    n = mb * 2**20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    reps = max(3, int(2048 / mb))
    s.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    h2d = n * reps / (s.elapsed_time(e) / 1e3) / 1e9
    s.record()
    for _ in range(reps):
        h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    d2h = n * reps / (s.elapsed_time(e) / 1e3) / 1e9
    res[mb] = (round(h2d, 2), round(d2h, 2))
out["h2d_d2h_GBs_by_MB"] = res
# 2 streams concurrent H2D
n = 256 * 2**20
hs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
ds = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(2)]
sts = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize()
t0 = time.perf_counter()
for r in range(8):
    for i in range(2):
        with torch.cuda.stream(sts[i]):
            ds[i].copy_(hs[i], non_blocking=True)
torch.cuda.synchronize()
out["h2d_2streams_GBs"] = 16 * n / (time.perf_counter() - t0) / 1e9
# pinned alloc speed
t0 = time.perf_counter()
big = torch.empty(8 * 2**30, dtype=torch.uint8, pin_memory=True)
out["pin_8GB_s"] = time.perf_counter() - t0
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/box_probe.json", "w"), indent=1)
