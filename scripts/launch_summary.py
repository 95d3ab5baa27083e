"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
tot = 0.0
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
    tot += v
print(f"total {tot/1e3:.1f} us over {sum(a[0] for a in agg.values())} launches")
print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {n} | {t/1e3:.1f} | {t/n/1e3:.2f} | {t/tot:.3f} |")
