"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel: launches, total, share."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in data:
    name = r[ki].split("(")[0].replace("void ", "")
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    us = v / 1000.0 if u in ("ns", "nsecond") else (v * 1000.0 if u in ("ms", "msecond") else v)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
print(f"# {sys.argv[1]}: {sum(a[0] for a in agg.values())} launches, {tot / 1000:.2f} ms total "
      "(ncu: cold caches, serialised — compare shares, not absolutes)")
print(f"{'kernel':58s} {'launches':>8s} {'total_ms':>9s} {'share':>6s} {'avg_us':>9s}")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:58]:58s} {c:8d} {t / 1000:9.3f} {100 * t / tot:5.1f}% {t / c:9.1f}")
