"""Device time of the thin QR's kernels (rtucker_qr, shifted CholeskyQR3) for an m x k fp64 matrix,
uncontended (main stream only): per-label times from the library's CUDA events.

    python tools/qr_time.py [--m 2048] [--ks 27 60 80 128] [--reps 5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_07124_b200 import _lib as L
from paper_2001_07124_b200 import api as P

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=2048)
ap.add_argument("--ks", type=int, nargs="+", default=[27, 60, 80, 128])
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
h = P.Handle()
for k in a.ks:
    Y = torch.randn(a.m, k, dtype=torch.float64, device="cuda")
    P.rtucker_qr(h, Y)
    h.sync()
    h.profile_read()
    h.set_option(L.RT_OPT_PROFILE, 1)
    for _ in range(a.reps):
        P.rtucker_qr(h, Y)
    h.sync()
    h.set_option(L.RT_OPT_PROFILE, 0)
    prof = h.profile_read()[0]
    print(f"k={k}: " + "  ".join(f"{n} {ms / a.reps * 1e3:.1f} us/{c // a.reps}" for n, c, ms in prof), flush=True)
