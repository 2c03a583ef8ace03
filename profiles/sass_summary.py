"""Per-kernel SASS opcode census of the shipped library (cuobjdump -sass): the
instructions that prove the tcgen05 / TMEM / TMA paths (UTCHMMA / UTCQMMA = tcgen05.mma,
LDTM = tcgen05.ld, UTMALDG = cp.async.bulk.tensor, UBLKCP = cp.async.bulk, LDGSTS =
cp.async) and the absence of legacy HMMA.  usage: python profiles/sass_summary.py > profiles/r2_sass_summary.md"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2111_01264_b200", "_lib", "libparaq_b200.so")
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "LDGSTS", "SYNCS", "HMMA",
       "DFMA", "FFMA"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
kernels = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kernels[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", line)
    if m:
        op = m.group(1)
        for o in OPS:
            if op == o or op.startswith(o + "."):
                kernels[cur][o] += 1


def short(name):
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    dem = re.sub(r"\bpq::", "", dem)
    return dem if len(dem) < 150 else dem[:147] + "..."


print(f"# SASS opcode census of {os.path.relpath(LIB, ROOT)}\n")
print("`cuobjdump -sass`, counts of static instructions per kernel (sm_100a).\n")
tot = collections.Counter()
for k, c in kernels.items():
    tot.update(c)
print("| totals | " + " | ".join(f"{o} {tot[o]}" for o in OPS if tot[o]) + " |\n")
print("| kernel | " + " | ".join(OPS) + " |")
print("|---" * (len(OPS) + 1) + "|")
for k, c in kernels.items():
    print(f"| `{short(k)}` | " + " | ".join(str(c[o]) if c[o] else "" for o in OPS) + " |")
