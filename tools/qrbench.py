"""Time rtucker_qr (sCQR3: gram, chol_inv, gemm_tall) on an m x k fp64 matrix, per kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2001_07124_b200 import _lib as L
from paper_2001_07124_b200 import api as P

m, k = int(sys.argv[1]) if len(sys.argv) > 1 else 2048, int(sys.argv[2]) if len(sys.argv) > 2 else 80
h = P.Handle()
Y = torch.randn((k, m), dtype=torch.float64, device="cuda").t()
for rep in range(3):
    h.set_option(L.RT_OPT_PROFILE, 1)
    Q, R = P.rtucker_qr(h, Y)
    h.sync()
    prof, n = h.profile_read()
    h.set_option(L.RT_OPT_PROFILE, 0)
    if rep:
        print(" ".join(f"{nm}:{c}x {1e3 * ms / c:.1f}us" for nm, c, ms in sorted(prof, key=lambda e: -e[2])))
