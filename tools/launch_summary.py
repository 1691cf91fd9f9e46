"""Summarise an ncu launch list (gpu__time_duration.sum CSV): per kernel+grid totals and shares.
    python tools/launch_summary.py launches.csv [by_grid]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
by_grid = len(sys.argv) > 2
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    k = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    if by_grid:
        k += " " + d["Grid Size"] + " " + d["Block Size"]
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"]) * scale.get(d["Metric Unit"], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':62s} {'launches':>8s} {'total us':>11s} {'share':>6s} {'avg us':>9s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:60]:
    print(f"{k:62s} {v[0]:8d} {v[1]:11.1f} {100 * v[1] / tot:5.1f}% {v[1] / v[0]:9.2f}")
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
