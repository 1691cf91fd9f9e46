"""Per-launch DRAM bytes of the roofline kernels from an ncu launch list, into
profiles/traffic.json (read by bench.py for roofline.traffic):

    python tools/traffic_from_ncu.py <launches.csv> <config> [source note]

The csv is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none --csv` of tools/prof_one.py on the
config's problem.  Kinds (bench.py PROFILE_KINDS): 0 finest colour pass
(k_bgs_inv, the largest-grid launches), 1 outer CSR SpMV (k_csr_spmv), 2
residual before restriction (k_rows, largest grid), 4 / 5 level-L down / up
visit (k_stream_down / k_stream_up or k_tile_down / k_tile_up, largest grid).
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KINDS = {0: ("k_bgs_inv(",), 1: ("k_csr_spmv",), 2: ("k_rows",), 4: ("k_stream_down", "k_tile_down"),
         5: ("k_stream_up", "k_tile_up")}


def main(path, cfg, note=""):
    launches = defaultdict(dict)
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"], d.get("Grid Size", ""))
        try:
            launches[key][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            pass
    out = {}
    for kind, names in KINDS.items():
        rows = []
        for nm in names:   # the first kernel family present (stream kernels before tiles)
            rows = [(k, m) for k, m in launches.items() if nm in k[1]]
            if rows:
                break
        if not rows:
            continue
        def grid(k):
            g = k[2].strip("()").split(",")
            return int(g[0]) if g and g[0].strip().isdigit() else 0
        gmax = max(grid(k) for k, _ in rows)
        sel = [m for k, m in rows if grid(k) == gmax]
        b = [m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in sel]
        out[str(kind)] = int(sum(b) / len(b))
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    data = json.load(open(tp)) if os.path.exists(tp) else {}
    data.setdefault(cfg, {}).update(out)
    if note:
        data["_source_" + cfg] = note
    json.dump(data, open(tp, "w"), indent=1)
    print(cfg, out)


if __name__ == "__main__":
    main(*sys.argv[1:4])
