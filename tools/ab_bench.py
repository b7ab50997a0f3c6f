"""A/B timing of RT_OPT_TC_ABLATE switches on one BASELINE config in ONE process (same box, same
clocks): the HOSVD step of bench.py, interleaved over the option values, CUDA events on the
handle's stream.

    python tools/ab_bench.py --config cfg5 --opts 270 271 --reps 5 [--profile]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from gen import synth
from paper_2001_07124_b200 import _lib as L
from paper_2001_07124_b200 import api as P

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--opts", type=int, nargs="+", required=True)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--profile", action="store_true", help="print the top kernel classes per option")
a = ap.parse_args()

cfg = synth.CONFIGS[a.config]
X, _ = synth.make_tensor_device(cfg, "cuda")
oms = [synth.gaussian_omega_device(cfg, n, "cuda", tf32=True) for n in range(cfg.order)]
stream = torch.cuda.Stream()
times = {o: [] for o in a.opts}
profs = {}
with torch.cuda.stream(stream):
    hs = {}
    for o in a.opts:
        h = P.Handle(stream=stream)
        h.set_option(L.RT_OPT_OMEGA_TF32, 1)
        h.set_option(100, o)
        P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms)      # warm-up (workspace)
        h.sync()
        hs[o] = h
    for rep in range(a.reps):
        for o in a.opts:
            h = hs[o]
            if a.profile and rep == a.reps - 1:
                h.profile_read()
                h.set_option(L.RT_OPT_PROFILE, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms)
            e1.record(stream)
            h.sync()
            times[o].append(e0.elapsed_time(e1))
            if a.profile and rep == a.reps - 1:
                h.set_option(L.RT_OPT_PROFILE, 0)
                profs[o] = sorted(h.profile_read()[0], key=lambda e: -e[2])
for o in a.opts:
    t = times[o]
    print(f"option {o}: median {statistics.median(t):.2f} ms  min {min(t):.2f}  all " +
          " ".join(f"{x:.2f}" for x in t), flush=True)
    if o in profs:
        print("   " + ", ".join(f"{n}:{c}x {ms:.2f}" for n, c, ms in profs[o][:14]))
