"""R-PET parity diagnostic: the oracle's E of the GPU factors/core vs the GPU's E vs the oracle's E."""
import sys, threading
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import oracle
from gen import synth
from paper_2001_07124_b200 import api as P

cfg = synth.CONFIGS["cfg5"].scaled((48, 40, 36), (6, 6, 6), (6, 6, 6))
x = synth.make_tensor(cfg)
ks, ss = synth.pet_sizes(cfg)
oms = [synth.gaussian_omega(cfg, n, K=ks[n]) for n in range(3)]
omt = [synth.omega_tilde(cfg, n, ss[n]) for n in range(3)]
ref = oracle.pet(x, cfg.ranks, oms, omt)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
h = P.Handle()
res = P.rtucker_pet(h, torch.from_numpy(synth.to_device_layout(x)).cuda(), cfg.ranks, [t(o) for o in oms], [t(o) for o in omt])
h.sync()
qg = [q.cpu().numpy() for q in res["Q"]]
gg = P.core_to_numpy(res["G"])
e_exact = oracle.rel_error(x, gg, qg)
print("oracle E", ref["E"], "gpu E", float(res["err"][0]), "exact E of gpu decomposition", e_exact)
print("rel(gpuE vs exact)", abs(float(res["err"][0]) - e_exact) / e_exact, "rel(exact vs oracle)", abs(e_exact - ref["E"]) / ref["E"])

from paper_2001_07124_b200 import _lib as L
for impl in (0, 1):
    h2 = P.Handle(); h2.set_option(L.RT_OPT_TTM_IMPL, impl)
    res = P.rtucker_pet(h2, torch.from_numpy(synth.to_device_layout(x)).cuda(), cfg.ranks, [t(o) for o in oms], [t(o) for o in omt])
    h2.sync()
    qg = [q.cpu().numpy() for q in res["Q"]]; gg = P.core_to_numpy(res["G"])
    ee = oracle.rel_error(x, gg, qg)
    print("pet impl", impl, "gpuE-exact", (float(res["err"][0]) - ee) / ee, "exact-oracle", (ee - ref["E"]) / ref["E"])
    # same factors/core through rtucker_core's E (projection core differs; only check residual eval)
    hs = P.rtucker_hosvd(h2, torch.from_numpy(synth.to_device_layout(x)).cuda(), cfg.ranks, cfg.p, cfg.q,
                         [t(synth.gaussian_omega(cfg, n)) for n in range(3)])
    h2.sync()
    qg = [q.cpu().numpy() for q in hs["Q"]]; gg = P.core_to_numpy(hs["G"])
    ee = oracle.rel_error(x, gg, qg)
    print("hosvd impl", impl, "gpuE-exact", (float(hs["err"][0]) - ee) / ee, "E", ee)
