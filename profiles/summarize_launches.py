"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in data:
    if len(r) <= vi:
        continue
    name = re.sub(r"\(.*", "", r[ki])
    m = re.search(r"k_gemm<(\d+), (\w+), (\w+), pq::(\w+), pq::(\w+), pq::(\w+)>", r[ki])
    if m:
        name = f"gemm BN{m.group(1)} {m.group(4)}/{m.group(5)}/{m.group(6)}"
    v = float(r[vi].replace(",", ""))
    v = v / 1000 if r[ui] in ("ns", "nsecond") else v * 1000 if r[ui] in ("ms", "msecond") else v
    agg[name].append(v)
tot = sum(sum(v) for v in agg.values())
print(f"{'share':>6} {'n':>5} {'avg us':>8}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v) / tot * 100:5.1f}% {len(v):5d} {sum(v) / len(v):8.2f}  {k}")
