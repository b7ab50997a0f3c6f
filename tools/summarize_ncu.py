"""Summarize ncu outputs into profiles/ (tracked):

    python tools/summarize_ncu.py --launches gpurun_out/launches.csv --full gpurun_out/prof.ncu-rep \
        --round r01 [--steps 2]

Writes profiles/<round>_launches.md (per-kernel-class device time and share of the step, from the
--metrics gpu__time_duration.sum launch list: cold-cache, serialised -> compare SHARES),
profiles/<round>_<kernel>_full.txt (key metrics of one --set full capture) and updates
profiles/traffic.json (DRAM bytes read+write per launch of the captured kernel, read by bench.py).
"""
import argparse
import csv
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel)", name)
    base = m.group(1) if m else name.split("(")[0]
    t = re.search(r"<([^>]*)>", name)
    return base + (f"<{t.group(1)}>" if t else "")


def launches(path, rnd):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    per = defaultdict(lambda: [0, 0.0])
    unit = "ns"
    ours = ("ttm_", "residual", "chol_inv", "jacobi", "gram_kernel", "gemm_tall", "gemm_small", "splitk", "reduce_p", "sumsq", "convert2d",
            "sign_apply", "colmax", "nonfinite", "split_transpose", "finalize_err", "unfold_copy", "loop_sum")
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        nm = d["Kernel Name"]
        if any(t in nm for t in ("at::", "c10::", "cub::", "cublas", "nccl")) or not (
                any(o in nm for o in ours) or "unnamed>::" in nm or "rt::" in nm):
            continue                        # torch's input-generation kernels (outside the timed region)
        unit = d.get("Metric Unit", unit)
        v = float(d["Metric Value"].replace(",", ""))
        k = short(d["Kernel Name"])
        per[k][0] += 1
        per[k][1] += v
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
    tot = sum(v[1] for v in per.values()) * scale
    lines = [f"# {rnd}: launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
             f"source: {os.path.relpath(path, ROOT)}; {sum(v[0] for v in per.values())} launches; "
             f"total {tot:.2f} ms of librtucker kernels (input generation by torch excluded; cold-cache, "
             "serialised: compare shares, not absolutes)", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {t * scale:.3f} | {100 * t * scale / tot:.1f}% |")
    out = os.path.join(PROF, f"{rnd}_launches.md")
    open(out, "w").write("\n".join(lines) + "\n")
    print(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second"]


def full(path, rnd):
    p = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(p.stdout.splitlines()))
    hdr, units = rows[0], rows[1]
    out_txt = []
    traffic = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = short(d.get("Kernel Name", "?"))
        out_txt.append(f"kernel: {d.get('Kernel Name', '?')}")
        for k in KEYS:
            if k in d:
                out_txt.append(f"  {k} = {d[k]} {u.get(k, '')}")
        def to_bytes(k):
            v = float(d[k].replace(",", ""))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u[k], 1)
            return v * mult
        if "dram__bytes_read.sum" in d:
            b = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
            traffic[name.split("<")[0].replace("_kernel", "")] = b
            out_txt.append(f"  traffic (dram read+write) = {b / 1e9:.3f} GB per launch")
    kname = list(traffic)[0] if traffic else "kernel"
    out = os.path.join(PROF, f"{rnd}_{kname}_full.txt")
    open(out, "w").write(f"# {rnd}: ncu --set full --clock-control none capture ({os.path.relpath(path, ROOT)})\n"
                         + "\n".join(out_txt) + "\n")
    tp = os.path.join(PROF, "traffic.json")
    cur = json.load(open(tp)) if os.path.exists(tp) else {}
    cur.update(traffic)
    cur["_source"] = f"{rnd}: {os.path.basename(path)}"
    json.dump(cur, open(tp, "w"), indent=1)
    print(out, traffic)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--round", default="r01")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, a.round)
    if a.full:
        full(a.full, a.round)
