"""Warp-stall samples of one kernel per source line: joins an ncu
`--page source --csv --print-source sass` export with `nvdisasm -g` line info
of the same cubin.   python tools/sass_lines.py <sass.csv> <nvdisasm.txt> <kernel-substring> [top]"""
import collections
import csv
import re
import sys


def line_map(path, kernel):
    m, cur, on = {}, None, False
    for ln in open(path):
        if ln.startswith("//---------------------"):
            on = kernel in ln and ".text." in ln
            continue
        if not on:
            continue
        f = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if f:
            cur = (f.group(1).split("/")[-1], int(f.group(2)))
            continue
        o = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+\S", ln)
        if o and cur:
            m[int(o.group(1), 16)] = cur
    return m


def main(csv_path, sass_path, kernel, top=40):
    lm = line_map(sass_path, kernel)
    rows = list(csv.reader(open(csv_path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    data = [r for r in rows if len(r) == len(hdr) and r[0].startswith("0x")]
    # the export may hold several launches of the kernel: one base per block of rows
    agg, reasons, total = collections.Counter(), collections.defaultdict(collections.Counter), collections.Counter()
    base = None
    for r in data:
        a = int(r[0], 16)
        if base is None or a < base:
            base = a
        off = a - base
        key = lm.get(off, ("?", 0))
        s = int(r[si] or 0)
        agg[key] += s
        for i in cols:
            v = int(r[i] or 0)
            reasons[key][hdr[i][6:]] += v
            total[hdr[i][6:]] += v
    T = sum(agg.values())
    print("samples", T)
    for k, v in total.most_common(8):
        print(f"  {k:20s} {v:7d} {100 * v / max(T, 1):5.1f}%")
    for key, v in agg.most_common(int(top)):
        print(f"{key[0]}:{key[1]:<5d} {v:6d} {100 * v / T:5.1f}%  ", dict(reasons[key].most_common(3)))


if __name__ == "__main__":
    main(*sys.argv[1:])
