"""Device time per call of the latency-bound kernel classes (Jacobi EVD, Cholesky, Gram, tall GEMM,
the R31' sample) from the library's own per-launch CUDA events (RT_OPT_PROFILE), on a cfg5-shaped
HOSVD (K = 80) and the cfg3 R-STHOSVD (Kronecker, K = 27).

    python tools/small_kernels.py [--dims 512 512 512] [--reps 3]
"""
import argparse
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from gen import synth
from paper_2001_07124_b200 import _lib as L
from paper_2001_07124_b200 import api as P

ap = argparse.ArgumentParser()
ap.add_argument("--dims", type=int, nargs=3, default=[512, 512, 512])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
CLASSES = ("jacobi_sweeps", "jacobi_eig", "chol_inv", "gram", "gemm_tall", "zsample", "unmix_cols", "splitk_reduce")


def show(tag, prof, reps):
    d = {n: (c, ms) for n, c, ms in prof}
    print(tag + "  " + "  ".join(f"{k} {d[k][1] / reps:.3f} ms/{d[k][0] // reps}" for k in CLASSES if k in d),
          flush=True)


cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled(tuple(a.dims), (64, 64, 64), (64, 64, 64)), p=16, q=1)
x = synth.make_tensor(cfg)
X = torch.from_numpy(synth.to_device_layout(x)).cuda()
oms = [torch.from_numpy(np.ascontiguousarray(synth.round_tf32(synth.gaussian_omega(cfg, n)))).cuda() for n in range(3)]
h = P.Handle()
h.set_option(L.RT_OPT_OMEGA_TF32, 1)
P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, 1, oms)
h.sync()
h.set_option(L.RT_OPT_PROFILE, 1)
for _ in range(a.reps):
    P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, 1, oms)
h.sync()
show(f"hosvd {tuple(a.dims)} K=80", h.profile_read()[0], a.reps)
h.close()

cfg = synth.CONFIGS["cfg3"]
x = synth.make_tensor(cfg)
X = torch.from_numpy(synth.to_device_layout(x)).cuda()
ko = [[None if o is None else torch.from_numpy(np.ascontiguousarray(synth.round_tf32(o))).cuda()
       for o in synth.kron_omegas(cfg, n, synth.sthosvd_dims_before(cfg, n))] for n in range(cfg.order)]
h = P.Handle()
h.set_option(L.RT_OPT_OMEGA_TF32, 1)
P.rtucker_sthosvd(h, X, cfg.ranks, cfg.p, cfg.q, ko, kind="kron")
h.sync()
h.set_option(L.RT_OPT_PROFILE, 1)
for _ in range(a.reps):
    P.rtucker_sthosvd(h, X, cfg.ranks, cfg.p, cfg.q, ko, kind="kron")
h.sync()
show("cfg3 sthosvd K=27", h.profile_read()[0], a.reps)
h.close()
