import dataclasses, numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
import oracle
from gen import synth
from tests import _metrics as M
from paper_2001_07124_b200 import api as P, _lib as L
for dims, rank, p in [((512, 384), 20, 12), ((512, 256, 48), 20, 12)]:
    N = len(dims)
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled(dims, (rank,) * N, (rank,) * N), p=p, q=1)
    x = synth.make_tensor(cfg)
    oms = [synth.round_tf32(synth.gaussian_omega(cfg, n)) for n in range(N)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    w = np.linalg.svd(oracle.unfold(ref["Gt"], 0), compute_uv=False)
    print(dims, "core sv 18..22:", w[17:23])
    for opt in (291, 290, 270):
        h = P.Handle(); h.set_option(L.RT_OPT_OMEGA_TF32, 1); h.set_option(100, opt)
        r = P.rtucker_hosvd(h, torch.from_numpy(synth.to_device_layout(x)).cuda(), cfg.ranks, cfg.p, 1,
                            [torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in oms])
        h.sync()
        print(opt, [f"{M.subspace(r['Q'][n].cpu().numpy(), ref['Q'][n]):.2e}" for n in range(N)],
              f"{abs(float(r['err'][0]) - ref['E'])/ref['E']:.2e}")
        h.close()
