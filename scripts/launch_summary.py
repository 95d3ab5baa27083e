"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,...] --csv`
launch list: time share per kernel (and DRAM bytes per launch when listed)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
agg = collections.OrderedDict()
tot = 0.0
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    a = agg.setdefault(name, {"n": 0, "us": 0.0, "bytes": 0.0})
    if r[mi] == "gpu__time_duration.sum":
        a["n"] += 1
        a["us"] += v
        tot += v
    elif r[mi].startswith("dram__bytes"):
        a["bytes"] += v
print(f"total {tot:.1f} us over {sum(a['n'] for a in agg.values())} launches")
print("| kernel | launches | total us | mean us | share | DRAM MB / launch |\n|---|---|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
    print(f"| {k} | {a['n']} | {a['us']:.1f} | {a['us'] / a['n']:.2f} | {a['us'] / tot:.3f} | {a['bytes'] / a['n'] / 1e6:.2f} |")
