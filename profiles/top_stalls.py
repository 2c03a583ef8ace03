"""Top SASS lines by warp-stall samples from `ncu -i X --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
samp = h.index("Warp Stall Sampling (All Samples)")
src = h.index("Source")
def num(x):
    try:
        return float(x)
    except ValueError:
        return None


body = [r for r in rows[2:] if len(r) > samp and num(r[samp]) is not None]
tot = sum(float(r[samp] or 0) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(body, key=lambda r: -float(r[samp] or 0))[:n]:
    print(f"{float(r[samp]) / tot * 100:5.1f}%  {r[0][-5:]}  {r[src].strip()[:90]}")
