"""Summarize an ncu --set full --import-source report: key metrics + warp-stall samples per SASS
instruction, aggregated by instruction opcode and by hot instructions.

    python tools/ncu_stalls.py gpurun_out/x.ncu-rep [--top 25]
"""
import argparse
import csv
import subprocess
import sys
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, d = rows[0], rows[1], rows[2]
print(d[h.index("Kernel Name")][:140])
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
          "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__registers_per_thread",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed"]:
    if k in h:
        print(f"  {k} = {d[h.index(k)]} {u[h.index(k)]}")
src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = None
data = []
for r in rows:
    if "Source" in r and "Address" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(x[key] or 0) for x in data)
by_op = defaultdict(float)
for x in data:
    op = x["Source"].strip().split()[0] if x["Source"].strip() else "?"
    if op.startswith("@"):
        op = x["Source"].strip().split()[1]
    by_op[op.split(".")[0]] += float(x[key] or 0)
print(f"stall samples total {tot:.0f}")
for op, v in sorted(by_op.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {op:20s} {100 * v / tot:5.1f}%")
print("hot instructions:")
for x in sorted(data, key=lambda x: -float(x[key] or 0))[:a.top]:
    print(f"  {100 * float(x[key] or 0) / tot:5.1f}%  {x['Address'][-5:]}  {x['Source'].strip()[:90]}")
