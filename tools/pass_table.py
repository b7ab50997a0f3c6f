"""Summarize tools/pass_table.sh output into profiles/<round>_passes.md: one row per X-streaming
launch of the timed step (ncu metrics; cold-cache, serialised -> compare with the bench's own
per-class timings for absolutes)."""
import csv
import os
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out", f"passes_{rnd}.csv")
rows = [r for r in csv.reader(open(src)) if r and r[0].isdigit()]
k = OrderedDict()
for r in rows:
    kid = int(r[0])
    d = k.setdefault(kid, {"name": r[4], "grid": r[8]})
    d[r[12]] = float(r[14].replace(",", ""))
launches = [v for v in k.values() if v.get("dram__bytes_read.sum", 0) > 20e9]   # X-streaming passes
half = len(launches) // 2
step = launches[half:]                                                      # timed step (after warmup)
out = [f"# {rnd}: per-pass ncu metrics of one cfg5 HOSVD step (`tools/pass_table.sh`)", "",
       "X-streaming launches only (DRAM read > 20 GB), in launch order.  `--clock-control none`,"
       " serialised, cold L2: shares and fractions are comparable, absolutes are slower than in the bench.", "",
       "| # | kernel | grid | ms | DRAM read GB | DRAM % of peak | tensor pipe % |", "|---|---|---|---|---|---|---|"]
for i, v in enumerate(step):
    nm = v["name"].replace("void unnamed>::", "").split("(")[0]
    out.append(f"| {i} | `{nm}` | {v['grid']} | {v.get('gpu__time_duration.sum', 0) / 1e6:.2f} | "
               f"{v.get('dram__bytes_read.sum', 0) / 1e9:.2f} | "
               f"{v.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
               f"{v.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f} |")
dst = os.path.join(ROOT, "profiles", f"{rnd}_passes.md")
open(dst, "w").write("\n".join(out) + "\n")
print(dst)
print("\n".join(out))
