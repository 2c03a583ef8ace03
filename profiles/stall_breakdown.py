"""Warp-stall reasons summed over a kernel's SASS (ncu --page source --csv --print-source sass),
and the top instructions with their dominant reason.  usage: stall_breakdown.py CSV [n]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
st = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
seen, tot, per = set(), Counter(), []
for r in rows[2:]:
    if len(r) < len(h) or r[0] in seen or r[0] == "Address":
        continue
    seen.add(r[0])
    c = Counter({h[i][6:]: float(r[i] or 0) for i in st})
    tot += c
    per.append((sum(c.values()), r[1].strip()[:70], c.most_common(2)))
s = sum(tot.values())
print("reasons:", ", ".join(f"{k} {v / s * 100:.1f}%" for k, v in tot.most_common(8)))
for n, src, top in sorted(per, key=lambda x: -x[0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{n / s * 100:5.1f}%  {src:70s} {', '.join(f'{k}:{v / s * 100:.1f}' for k, v in top)}")
