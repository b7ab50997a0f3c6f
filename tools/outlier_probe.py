"""Probe: cfg2-small HOSVD (q = 1) with three entries A times max|bulk| (three extra rank-1 terms),
tf32 kernels (RT_OPT_TC_ABLATE 210) vs the fp16 split (211), subspace distance to the oracle and E.
Measured (r01): A = 1e3 gives identical results on both paths (E = 3e-7 vs the oracle's 1e-8: E
relative to an outlier-dominated ||X|| is below fp32 resolution); A = 1e5 breaks the CholeskyQR on
both.  Such data are outside the fp32 path whatever the split (R29).

    python tools/outlier_probe.py
"""
import sys, numpy as np, torch, dataclasses
sys.path.insert(0, ".")
from gen import synth
import oracle
from paper_2001_07124_b200 import api as P
from tests import _metrics as M
for A, R in ((1e3, 23), (1e3, 20), (1e5, 23)):
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"].scaled((200, 180, 160), (20, 20, 20), (R, R, R)), p=32 - R)
    x = synth.make_tensor(cfg).astype(np.float64)
    rng = np.random.default_rng(12)
    for _ in range(3):
        idx = tuple(int(rng.integers(0, d)) for d in x.shape); x[idx] = A * np.abs(x).max()
    x = np.asfortranarray(x.astype(np.float32))
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    for ab in (210, 211):
        h = P.Handle(); h.set_option(100, ab)
        try:
            res = P.rtucker_hosvd(h, torch.from_numpy(synth.to_device_layout(x)).cuda(), cfg.ranks, cfg.p, 1, [torch.from_numpy(o).cuda() for o in oms]); h.sync()
            print(A, R, ab, ["%.2e" % M.subspace(q.cpu().numpy(), ref["Q"][n]) for n, q in enumerate(res["Q"])], float(res["err"][0]), ref["E"], flush=True)
        except Exception as e:
            print(A, R, ab, "ERR", e, flush=True)
        h.close()
