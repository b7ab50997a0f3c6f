"""Accumulation-precision probe of the tcgen05 sketch vs SIMT vs fp64 (long contraction)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from gen import synth
from paper_2001_07124_b200 import api as P, _lib as L

dims = (256, 1024, 1024)
x = np.asfortranarray(np.random.default_rng(5).standard_normal(dims).astype(np.float32))
X = torch.from_numpy(synth.to_device_layout(x)).cuda()
for n in (0, 2):
    J = x.size // dims[n]
    om = np.random.default_rng(6).standard_normal((J, 80)).astype(np.float32)
    omd = torch.from_numpy(om).cuda()
    y0 = oracle.unfold(x.astype(np.float64), n) @ om.astype(np.float64)
    for impl, seg in [(1, 0), (2, 1), (2, 4), (2, 32), (2, 128), (2, 100000)]:
        h = P.Handle()
        h.set_option(L.RT_OPT_TTM_IMPL, impl)
        if seg: h.set_option(L.RT_OPT_TC_SEGMENT, seg)
        y = P.rtucker_sketch(h, X, n, omd).cpu().numpy()
        h.sync()
        e = np.linalg.norm(y - y0) / np.linalg.norm(y0)
        print(f"mode {n} impl {impl} seg {seg}: rel err {e:.3e}", flush=True)
        h.close()
