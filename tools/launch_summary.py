"""Summarise an ncu launch list (CSV with gpu__time_duration.sum and optionally
dram__bytes_read.sum / dram__bytes_write.sum): per kernel (+grid) launches,
total time, share, average time, average DRAM bytes and GB/s.
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
tscale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
bscale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}
per = collections.defaultdict(dict)   # launch ID -> fields
for d in data:
    k = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    if by_grid:
        k += " " + d["Grid Size"]
    e = per[d["ID"]]
    e["k"] = k
    m, v, u = d["Metric Name"], float(d["Metric Value"].replace(",", "")), d["Metric Unit"]
    if m == "gpu__time_duration.sum":
        e["t"] = v * tscale.get(u, 1.0)
    elif m.startswith("dram__bytes"):
        e["b"] = e.get("b", 0.0) + v * bscale.get(u, 1.0)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for e in per.values():
    a = agg[e["k"]]
    a[0] += 1
    a[1] += e.get("t", 0.0)
    a[2] += e.get("b", 0.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':46s} {'launches':>8s} {'total us':>10s} {'share':>6s} {'avg us':>9s} {'avg MB':>8s} {'GB/s':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:45]:
    gbs = v[2] / (v[1] * 1e3) if v[1] else 0.0
    print(f"{k[:46]:46s} {v[0]:8d} {v[1]:10.1f} {100 * v[1] / tot:5.1f}% {v[1] / v[0]:9.2f} {v[2] / v[0] / 1e6:8.2f} {gbs:7.0f}")
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
