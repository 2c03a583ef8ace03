"""Per-kernel table + traffic JSON from an `ncu --set full` capture of one learner step.
usage: python profiles/ncu_step_summary.py REP.ncu-rep OUT_TRAFFIC.json [source-note]
Prints a markdown table (kernel, grid, us, DRAM MB, tensor pipe %, IPC)."""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed.avg.per_cycle_active", "launch__grid_size"]
SCALE = {"usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
         "Gbyte": 1e9, "": 1.0}

rep, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
head, units = rows[0], rows[1]
kernels = []
for r in rows[2:]:
    d = dict(zip(head, r))
    name = re.sub(r"^void (pq::)?", "", d["Kernel Name"]).replace("pq::", "")
    name = re.sub(r"\(.*\)$", "", name)
    k = {"name": name}
    for m in METRICS:
        i = head.index(m)
        v = float(r[i].replace(",", "")) if r[i] else 0.0
        k[m] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
    kernels.append(k)
dram = sum(k["dram__bytes_read.sum"] + k["dram__bytes_write.sum"] for k in kernels)
serial = sum(k["gpu__time_duration.sum"] for k in kernels)
json.dump({"source": note, "learner_step_dram_bytes": dram, "learner_step_serial_us": round(serial, 1),
           "launches": len(kernels), "kernels": kernels}, open(out, "w"), indent=1)
print("| kernel | grid | us (cold) | DRAM read+write MB | tensor pipe % | IPC |")
print("|---|---|---|---|---|---|")
for k in kernels:
    short = k["name"] if len(k["name"]) < 120 else k["name"][:117] + "..."
    print(f"| `{short}` | {int(k['launch__grid_size'])} | {k['gpu__time_duration.sum']:.1f} | "
          f"{(k['dram__bytes_read.sum'] + k['dram__bytes_write.sum']) / 1e6:.2f} | "
          f"{k['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']:.1f} | "
          f"{k['sm__inst_executed.avg.per_cycle_active']:.2f} |")
print(f"\nOne step: {len(kernels)} launches, {dram / 1e6:.1f} MB of DRAM traffic, {serial:.1f} us serialised cold.")
