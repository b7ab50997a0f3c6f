"""One cfg5 HOSVD call with RT_OPT_TC_ABLATE = argv[1] (0 = none, 1 = no MMA, 2 = no split work;
results invalid under an ablation) for ncu timing of the X-pass kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from gen import synth
from paper_2001_07124_b200 import _lib as L
from paper_2001_07124_b200 import api as P

ab = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = synth.CONFIGS["cfg5"]
X, _ = synth.make_tensor_device(cfg, "cuda")
oms = [synth.gaussian_omega_device(cfg, n, "cuda", tf32=True) for n in range(cfg.order)]
h = P.Handle()
h.set_option(L.RT_OPT_OMEGA_TF32, 1)
P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms)
h.sync()
if ab:
    h.set_option(L.RT_OPT_TC_ABLATE, ab)
try:
    P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms)
    h.sync()
except Exception as e:          # an ablated run may fail its numeric checks
    print("ablated call:", e)
