"""Diagnostic: cfg3 full STHOSVD (Kronecker) GPU vs oracle metrics, per TTM implementation."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from gen import synth
from paper_2001_07124_b200 import api as P
from tests import _metrics as M

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = synth.CONFIGS[name]
x = synth.make_tensor(cfg)
N = cfg.order
if cfg.algo == "sthosvd":
    oms = [synth.kron_omegas(cfg, n, synth.sthosvd_dims_before(cfg, n)) for n in range(N)]
    ref = oracle.sthosvd(x, cfg.ranks, oms, q=cfg.q, kind="kron")
else:
    oms = [synth.round_tf32(synth.gaussian_omega(cfg, n)) for n in range(N)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=cfg.q)
X = torch.from_numpy(synth.to_device_layout(x)).cuda()
print("oracle E", ref["E"], "E_gram", ref["E_gram"])
for impl in (0, 1):
    h = P.Handle()
    h.set_option(0, impl)
    h.set_option(3, 1)
    if cfg.algo == "sthosvd":
        dom = [[None if o is None else torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in row] for row in oms]
        res = P.rtucker_sthosvd(h, X, cfg.ranks, cfg.p, cfg.q, dom, kind="kron")
    else:
        res = P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, [torch.from_numpy(o).cuda() for o in oms])
    h.sync()
    qg = [q.cpu().numpy() for q in res["Q"]]
    gg = P.core_to_numpy(res["G"])
    e = res["err"].cpu().numpy()
    print(f"impl {impl}: M2", [f"{M.subspace(q, ref['Q'][n]):.2e}" for n, q in enumerate(qg)],
          f"M4 {M.core_in_oracle_basis(gg, qg, ref['G'], ref['Q']):.2e} M5 {M.recon(gg, qg, ref['G'], ref['Q']):.2e}",
          f"E {e[0]:.10e} relerr {abs(e[0] - ref['E']) / ref['E']:.2e} E_gram {e[1]:.6e}",
          f"|G| {np.linalg.norm(gg):.10e} vs {np.linalg.norm(ref['G']):.10e}")
    # E implied by the GPU's own factors, computed by the oracle
    e_o = oracle.rel_error(x, gg, qg)
    print(f"   oracle E of GPU factors {e_o:.10e} relerr vs GPU E {abs(e[0] - e_o) / e_o:.2e}")
    h.close()
