"""Summarise an ncu --csv metrics log of warp-stall ratios: per kernel (first launch of
each name), the stall reasons sorted by cycles per issued instruction.

    python tools/stall_summary.py gpurun_out/stalls/stalls_c6.csv
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
per = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    key = (d["ID"], d["Kernel Name"].split("(")[0])
    try:
        v = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    per.setdefault(key, {})[d["Metric Name"]] = v
out = {}
for (i, k), m in per.items():
    if k in out:
        continue
    st = {n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): round(v, 2)
          for n, v in m.items() if "stalled" in n and v >= 0.05}
    out[k] = {"us": m.get("gpu__time_duration.sum"), "warps_active_pct": m.get("smsp__warps_active.avg.pct_of_peak_sustained_active"),
              "dram_pct": m.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
              "stalls_per_issue": dict(sorted(st.items(), key=lambda kv: -kv[1]))}
print(json.dumps(out, indent=1))
