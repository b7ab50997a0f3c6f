import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, dataclasses
import oracle
from gen import synth
from paper_2001_07124_b200 import api as P, _lib as L
cfg = dataclasses.replace(synth.CONFIGS["cfg3"].scaled((34, 32, 30, 28), (5, 5, 5, 5), (5, 5, 5, 5)), q=1)
x = synth.make_tensor(cfg)
X = torch.from_numpy(synth.to_device_layout(x)).cuda()
oms = [synth.kron_omegas(cfg, n, cfg.dims) for n in range(4)]
for impl in (1, 0):
    h = P.Handle(); h.set_option(L.RT_OPT_TTM_IMPL, impl)
    for n in range(4):
        om = [None if o is None else torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in oms[n]]
        for q in (0, 1):
            try:
                y = P.rtucker_sketch(h, X, n, om, q=q, kind="kron").cpu().numpy()
                h.sync()
                _, yo = oracle.sketch_kron(x, n, oms[n], q)
                qa = np.linalg.qr(y)[0]; qb = np.linalg.qr(yo)[0]
                print(impl, n, q, "ok", np.linalg.norm(qa @ qa.T - qb @ qb.T))
            except Exception as e:
                print(impl, n, q, "ERR", e)
    h.close()
# Z-QR directly: qr of a fp32 tall matrix via rtucker_qr? (fp64 path) -> test TC gram on Z-like
