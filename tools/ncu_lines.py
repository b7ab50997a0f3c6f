"""Warp-stall samples of one kernel in an ncu --set full report, per CUDA source line: the SASS page's
per-instruction samples mapped to lines through nvdisasm -g of the kernel's cubin.

    python tools/ncu_lines.py gpurun_out/x.ncu-rep <cubin> <mangled-name-substring> [--launch 0] [--top 30]
"""
import argparse
import csv
import re
import subprocess
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("cubin")
ap.add_argument("name")
ap.add_argument("--launch", type=int, default=0)
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()
src = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip",
                      str(a.launch), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr, data = None, []
for r in rows:
    if "Source" in r and "Address" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
key = "Warp Stall Sampling (All Samples)"
addr = [int(x["Address"], 16) for x in data]
base = min(addr)
dis = subprocess.run(["nvdisasm", "-gi", a.cubin], capture_output=True, text=True).stdout.splitlines()
line_of, cur, inside = {}, None, False
for ln in dis:
    if ln.startswith(".text.") and a.name in ln:
        inside = True
        continue
    if inside and ln.startswith("//----------------"):
        if line_of:
            break
    if not inside:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', ln)
    if "//## File" in ln and m:
        # an inlined helper is charged to its call site in the kernel (the outermost "inlined at")
        cur = (m.group(3), int(m.group(4))) if m.group(3) else (m.group(1), int(m.group(2)))
    m2 = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m2 and cur is not None:
        line_of[int(m2.group(1), 16)] = cur
tot = sum(float(x[key] or 0) for x in data)
by_line = defaultdict(float)
for x, ad in zip(data, addr):
    by_line[line_of.get(ad - base, ("?", 0))] += float(x[key] or 0)
texts = {}
print(f"stall samples {tot:.0f}")
for (fn, ln), v in sorted(by_line.items(), key=lambda kv: -kv[1])[:a.top]:
    if fn not in texts:
        try:
            texts[fn] = open(fn).read().splitlines()
        except OSError:
            texts[fn] = []
    t = texts[fn]
    s = t[ln - 1].strip()[:96] if 0 < ln <= len(t) else "?"
    print(f"{100 * v / tot:5.1f}%  {fn.split('/')[-1]}:{ln}: {s}")
