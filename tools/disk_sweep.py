"""Disk-tier probe (SURVEY.md §8(d) nvme_probe; App. A / Fig. 6 analogue):
O_DIRECT read bandwidth of 4 GiB of blob-like files for reader threads x request size.
Writes the files under the given directory (default /tmp/pipo_disk_probe) once."""
import json
import os
import sys

sys.path.insert(0, ".")
from bench import disk_probe  # noqa: E402

d = sys.argv[1] if len(sys.argv) > 1 else "/tmp/pipo_disk_probe"
os.makedirs(d, exist_ok=True)
per, nfiles = 256 << 20, 16
blk = os.urandom(1 << 20)
for i in range(nfiles):
    p = os.path.join(d, f"layer_{i}.pipo")
    if not os.path.exists(p) or os.path.getsize(p) != per:
        with open(p, "wb") as f:
            for _ in range(per >> 20):
                f.write(blk)
os.sync()
out = {}
for threads in (1, 2, 4, 8, 16):
    for mb in (1, 4, 8, 16, 32, 64):
        out[f"t{threads}_b{mb}MiB"] = round(disk_probe(d, threads, mb << 20), 2)
        print(threads, mb, out[f"t{threads}_b{mb}MiB"], flush=True)
json.dump(out, open("gpurun_out/disk_sweep.json", "w"), indent=1)
