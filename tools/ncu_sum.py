"""Summarise an `ncu --csv --metrics gpu__time_duration.sum` launch list from stdin: per-kernel count and mean."""
import collections
import csv
import sys

rows = [r for r in csv.reader(sys.stdin) if len(r) > 5]
if not rows:
    sys.exit(0)
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1.0)
    a = agg.setdefault(r[ki][:60], [0, 0.0])
    a[0] += 1
    a[1] += v
for k, (c, t) in agg.items():
    print(f"{c:4d} x {t / c:8.4f} ms  {k}")
