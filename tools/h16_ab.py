"""A/B of the fp16-split kernels (RT_OPT_TC_ABLATE 210 = off, 211 = on) on the cfg5 HOSVD step:
per-label device times from the library's CUDA-event profiler.

    python tools/h16_ab.py [--reps 2]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from gen import synth  # noqa: E402
from paper_2001_07124_b200 import _lib as L  # noqa: E402
from paper_2001_07124_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--cfg", default="cfg5")
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
X, _ = synth.make_tensor_device(cfg, "cuda")
oms = [torch.from_numpy(synth.round_tf32(synth.gaussian_omega(cfg, n))).cuda() for n in range(cfg.order)]
h = api.Handle()
h.set_option(L.RT_OPT_OMEGA_TF32, 1)
for ab in (210, 211, 210, 211):
    h.set_option(L.RT_OPT_TC_ABLATE, ab)
    for rep in range(a.reps):
        h.set_option(L.RT_OPT_PROFILE, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h.stream)
        api.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms)
        e1.record(h.stream)
        h.sync()
        torch.cuda.synchronize()
        prof, _ = h.profile_read()
        h.set_option(L.RT_OPT_PROFILE, 0)
        if rep == 0:
            continue
        prof.sort(key=lambda e: -e[2])
        top = ", ".join(f"{nm}:{c}x{ms / c:.2f}" for nm, c, ms in prof[:7])
        print(f"h16={ab == 211} total {e0.elapsed_time(e1):.1f} ms: {top}", flush=True)
h.close()
