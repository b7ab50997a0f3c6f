"""Per-launch table of one library call from an ncu CSV (--metrics gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum[, ...]): the librtucker launches of the LAST call in the
capture (a warm-up call first), in launch order, with the bytes-per-time roofline of each.

    python tools/launch_table.py gpurun_out/cfg3_launches.csv --calls 2 --title "..." > profiles/x.md
"""
import argparse
import collections
import csv
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    by = collections.OrderedDict()
    for d in data:
        e = by.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [v for v in by.values() if "rt::" in v["name"]]


def short(name):
    n = re.sub(r"\(.*", "", name).replace("void ", "").replace("rt::<unnamed>::", "").replace("rt::", "")
    return n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--calls", type=int, default=2, help="library calls in the capture (the last is tabled)")
    ap.add_argument("--title", default="")
    ap.add_argument("--min-us", type=float, default=0.0)
    a = ap.parse_args()
    L = load(a.csv)
    per = len(L) // a.calls
    call = L[len(L) - per:]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    tot = sum(l["gpu__time_duration.sum"] for l in call) / 1e6
    print(f"# {a.title}\n")
    print(f"source: `{os.path.basename(a.csv)}` (ncu --clock-control none, serialised, cold L2); {len(call)} "
          f"librtucker launches in the timed call, {tot:.3f} ms summed.  `GB/s` = (DRAM read + write) / "
          f"launch time; `frac` against the measured copy peak {peak:.0f} GB/s.\n")
    print("| # | kernel | grid | us | DRAM rd MB | DRAM wr MB | GB/s | frac |")
    print("|---|---|---|---|---|---|---|---|")
    cls = collections.defaultdict(float)
    for i, l in enumerate(call):
        t = l["gpu__time_duration.sum"] / 1e3
        cls[short(l["name"]).split("<")[0]] += t
        if t < a.min_us:
            continue
        rd, wr = l.get("dram__bytes_read.sum", 0) / 1e6, l.get("dram__bytes_write.sum", 0) / 1e6
        gbs = (rd + wr) / 1e3 / (t / 1e6) if t else 0
        print(f"| {i} | `{short(l['name'])}` | {l['grid']} | {t:.1f} | {rd:.1f} | {wr:.1f} | {gbs:.0f} | {gbs / peak:.2f} |")
    print("\n| kernel class | us | share |")
    print("|---|---|---|")
    for k, v in sorted(cls.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {v:.1f} | {v / (tot * 1e3):.1%} |")


if __name__ == "__main__":
    main()
