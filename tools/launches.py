"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        n = d["Kernel Name"].split("(")[0].replace("void ", "").replace("pkv::<unnamed>::", "")[:48]
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"]) / (1e6 if d["Metric Unit"] == "ns" else 1e3)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tot = sum(v for _, v in agg.values())
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c // steps:5d} launches  {v / steps:9.3f} ms/step  {100 * v / tot:5.1f}%  {n}")
print(f"total {tot / steps:.3f} ms/step")
