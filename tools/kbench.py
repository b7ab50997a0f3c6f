"""Per-kernel timing of the hot TTM kernels through the C-ABI (CUDA events in librtucker).

    python tools/kbench.py --dims 2048 2048 2048 --K 80 --what sketch --reps 3 [--impl 2] [--seg 4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2001_07124_b200 import _lib as L
from paper_2001_07124_b200 import api as P

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs="+", default=[2048, 2048, 2048])
ap.add_argument("--K", type=int, default=80)
ap.add_argument("--what", default="sketch", choices=["sketch", "power", "core"])
ap.add_argument("--modes", type=int, nargs="*", default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--impl", type=int, default=0)
ap.add_argument("--seg", type=int, default=0)
ap.add_argument("--tf32", type=int, default=0)
ap.add_argument("--ablate", type=int, default=0)
ap.add_argument("--skew", type=int, default=-1)
ap.add_argument("--synth", default="", help="take X from gen.synth.make_tensor_device(CONFIGS[name]) instead of randn")
a = ap.parse_args()

dims = a.dims
N = len(dims)
if a.synth:
    from gen import synth
    X = synth.make_tensor_device(synth.CONFIGS[a.synth], "cuda")[0]
    dims = synth.CONFIGS[a.synth].dims
    N = len(dims)
else:
    X = torch.randn(tuple(reversed(dims)), device="cuda", dtype=torch.float32)
xbytes = X.numel() * 4
h = P.Handle()
h.set_option(L.RT_OPT_TTM_IMPL, a.impl)
h.set_option(L.RT_OPT_OMEGA_TF32, a.tf32)
if a.seg:
    h.set_option(L.RT_OPT_TC_SEGMENT, a.seg)
if a.ablate:
    h.set_option(100, a.ablate)
if a.skew >= 0:
    h.set_option(L.RT_OPT_TC_SKEW, a.skew)
modes = range(N) if a.modes is None else a.modes
for n in modes:
    J = X.numel() // dims[n]
    om = torch.randn((J, a.K), device="cuda", dtype=torch.float32)
    if a.tf32:
        om = (om.view(torch.int32) & -8192).view(torch.float32)
    qs = [torch.linalg.qr(torch.randn((d, a.K), device="cuda", dtype=torch.float64))[0] for d in dims]
    for rep in range(a.reps + 1):
        h.set_option(L.RT_OPT_PROFILE, 1)
        if a.what == "sketch":
            P.rtucker_sketch(h, X, n, om)
        elif a.what == "power":
            P.rtucker_sketch(h, X, n, om, q=1)
        else:
            P.rtucker_core(h, X, qs, with_error=False)
        h.sync()
        prof, launches = h.profile_read()
        h.set_option(L.RT_OPT_PROFILE, 0)
        if rep == 0:
            continue
        prof.sort(key=lambda e: -e[2])
        top = ", ".join(f"{nm}:{c}x {ms:.3f}ms ({xbytes * c / (ms * 1e-3) / 1e9:.0f} GB/s/launch-X)"
                        for nm, c, ms in prof[:4])
        print(f"mode {n} rep {rep}: {top}", flush=True)
    if a.what == "core":
        break
h.close()
