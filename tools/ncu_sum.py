"""Summarise ncu --csv launch lists: per kernel, launches and mean duration / DRAM bytes."""
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, agg, order = None, {}, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = d["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0]
            key = (k, d["Metric Name"])
            if key not in agg:
                agg[key] = []
                order.append(key)
            agg[key].append(float(d["Metric Value"].replace(",", "")))
    print("==", path)
    for key in order:
        v = agg[key]
        print(f"  {key[0]:28s} {key[1]:28s} n={len(v):3d} mean={sum(v) / len(v):.5g}")
