"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`.

    python tools/sass_hot.py /tmp/x_sass.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
tot = 0
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    n = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot += n
    st = sorted(((float(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    data.append((n, r[ix["Address"]], r[ix["Source"]], r[ix["Instructions Executed"]], st))
data_sorted = sorted(data, key=lambda t: -t[0])
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot)
for n, a, s, ie, st in data_sorted[:top]:
    print(f"{n / tot * 100:5.1f}% {a} {s[:60]:60s} exec={ie} " + " ".join(f"{c}:{v:.0f}" for v, c in st if v))
