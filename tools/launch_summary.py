"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: mean us per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = None
out = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if h is None or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
    out.setdefault(d["Kernel Name"][:70], []).append(v)
tot = 0.0
for k, v in out.items():
    print(f"{len(v):4d} x {sum(v) / len(v):9.1f} us  {k}")
