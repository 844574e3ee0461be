"""Summarise ncu output for profiles/: per-kernel launch-list aggregates (from a
`--metrics gpu__time_duration.sum --csv` log) and per-launch DRAM traffic / throughput
counters (from a `--set full` .ncu-rep via `ncu -i ... --page raw --csv`).

    python tools/ncu_summary.py launches gpurun_out/X/ncu_launches_c5.csv > profiles/.../launches_summary.json
    python tools/ncu_summary.py full gpurun_out/X/prof_c5_decode.ncu-rep > profiles/.../ncu_full_summary.json
"""
import collections
import csv
import io
import json
import subprocess
import sys

_SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
          "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def _num(v, unit):
    return float(v.replace(",", "")) * _SCALE.get(unit, 1.0)


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += _num(d["Metric Value"], d["Metric Unit"])
    tot = sum(v[1] for v in agg.values())
    out = {k: {"launches": n, "total_us": round(t, 2), "avg_us": round(t / n, 2), "share": round(t / tot, 4)}
           for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])}
    return {"source": path, "note": "ncu --clock-control none, serialised cold-cache launches", "total_us": round(tot, 1),
            "kernels": out}


FULL_METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
                "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
                "gpc__cycles_elapsed.max", "smsp__cycles_active.avg"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        e = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for m in FULL_METRICS:
            if m in h:
                i = h.index(m)
                try:
                    e[m] = _num(r[i], units[i])
                except ValueError:
                    e[m] = r[i]
        if "dram__bytes_read.sum" in e:
            e["traffic_bytes"] = e["dram__bytes_read.sum"] + e.get("dram__bytes_write.sum", 0.0)
            e["dram_gbs"] = e["traffic_bytes"] / (e["gpu__time_duration.sum"] * 1e-6) / 1e9
        res.append(e)
    return {"source": path, "note": "ncu --set full --clock-control none (cold cache, replayed)", "launches": res}


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if mode == "launches" else full(path), indent=1))
