"""One rank's share of the slab-parallel cfg5 step at P = 1, 2, 4, 8 ranks, timed on ONE GPU.

Only one GPU is available to this build, and ranks whose kernels wait on one another must not be
emulated on it.  What can be measured is the device time of rank 0's own work: its slab of X
(I_3 / P frontal slices), its rows of Omega_1 / Omega_2 and the whole Omega_3, through the
distributed code path of the library (a 1-rank NCCL communicator with RT_OPT_FORCE_COLLECTIVES: every
C1-C5 exchange is issued, each costing a 1-rank NCCL launch).  The P-rank step time is then this
plus the NVLink time of the exchanges that are not overlapped (DESIGN.md §7 gives their sizes).

    python tools/rank_share.py [--ranks 1 2 4 8] [--reps 5] [--profile]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from gen import synth
from paper_2001_07124_b200 import _lib as L
from paper_2001_07124_b200 import api as P
from paper_2001_07124_b200 import partition

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--opt", type=int, default=0, help="RT_OPT_TC_ABLATE value")
ap.add_argument("--profile", action="store_true")
ap.add_argument("--out", default=None)
a = ap.parse_args()

cfg = synth.CONFIGS[a.config]
N = cfg.order
I_last = cfg.dims[-1]
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
rows = []
with torch.cuda.stream(stream):
    for world in a.ranks:
        lo, hi = partition.slab_range(I_last, world, 0)
        X, _ = synth.make_tensor_device(cfg, dev, last_range=(lo, hi))
        oms = []
        for n in range(N):
            r = partition.omega_rows(cfg.dims, n, lo, hi)
            if r is not None:
                oms.append(synth.gaussian_omega_device(cfg, n, dev, row0=r[0], rows=r[1], tf32=True))
            else:
                oms.append(synth.gaussian_omega_device(cfg, n, dev, tf32=True))
        torch.cuda.synchronize()
        if world > 1:
            h = P.Handle(stream=stream, nccl_id=P.get_unique_id(), nranks=1, rank=0)
            h.set_option(L.RT_OPT_FORCE_COLLECTIVES, 1)
        else:
            h = P.Handle(stream=stream)
        h.set_option(L.RT_OPT_OMEGA_TF32, 1)
        if a.opt:
            h.set_option(100, a.opt)

        def step():
            return P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms, last_offset=lo, last_global=I_last)

        for _ in range(3):
            res = step()
        h.sync()
        ts = []
        prof = None
        for rep in range(a.reps):
            last = a.profile and rep == a.reps - 1
            if last:
                h.profile_read()
                h.set_option(L.RT_OPT_PROFILE, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = step()
            e1.record(stream)
            h.sync()
            ts.append(e0.elapsed_time(e1))
            if last:
                h.set_option(L.RT_OPT_PROFILE, 0)
                prof = sorted(h.profile_read()[0], key=lambda e: -e[2])
        E = float(res["err"][0].item())
        row = {"ranks": world, "slab": [lo, hi], "ms_median": statistics.median(ts), "ms_min": min(ts),
               "ms_all": [round(t, 3) for t in ts], "rel_err": E}
        if prof:
            row["kernels"] = [{"name": e[0], "count": e[1], "ms": round(e[2], 3)} for e in prof[:14]]
        rows.append(row)
        print(json.dumps(row), flush=True)
        h.close()
        del X, oms, res
        torch.cuda.empty_cache()
t1 = next((r["ms_median"] for r in rows if r["ranks"] == 1), None)
if t1:
    for r in rows:
        print(f"P = {r['ranks']}: rank share {r['ms_median']:.2f} ms, T_1 / share = {t1 / r['ms_median']:.2f}")
if a.out:
    with open(a.out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
