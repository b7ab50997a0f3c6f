"""Precision diagnosis: per-mode subspace distance to the oracle of one HOSVD case under the
RT_OPT_TC_ABLATE switches (212 tf32 twins, 240 QR of Z, 250 fp32 Omega sketches, 270 no overlap)
and the strict fp64 mode (TTM_IMPL 3).  Usage: python tools/prec_diag.py [case ...]"""
import dataclasses
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle  # noqa: E402
from gen import synth  # noqa: E402
from paper_2001_07124_b200 import _lib as L, api as P  # noqa: E402
from tests import _metrics as M  # noqa: E402

CASES = {
    "o2": (synth.CONFIGS["cfg2"], (300, 200), 12, 12, 1),
    "o2b": (synth.CONFIGS["cfg2"], (320, 256), 12, 12, 1),
    "o3": (synth.CONFIGS["cfg2"], (120, 110, 100), 10, 10, 1),
}
VARIANTS = [("default", []), ("212 twins", [(L.RT_OPT_TC_ABLATE, 212)]),
            ("240 qrz", [(L.RT_OPT_TC_ABLATE, 240)]), ("250 om32", [(L.RT_OPT_TC_ABLATE, 250)]),
            ("270 no-ovl", [(L.RT_OPT_TC_ABLATE, 270)]), ("strict", [(L.RT_OPT_TTM_IMPL, 3)])]


def main():
    names = sys.argv[1:] or list(CASES)
    for name in names:
        base, dims, r, p, q = CASES[name]
        N = len(dims)
        cfg = dataclasses.replace(base.scaled(dims, (r,) * N, (r,) * N), p=p, q=q)
        x = synth.make_tensor(cfg)
        oms = [synth.gaussian_omega(cfg, n) for n in range(N)]
        ref = oracle.hosvd(x, cfg.ranks, oms, q=q)
        X = torch.from_numpy(synth.to_device_layout(x)).cuda()
        for vname, opts in VARIANTS:
            h = P.Handle()
            for o, v in opts:
                h.set_option(o, v)
            res = P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, q, [torch.from_numpy(np.ascontiguousarray(o)).cuda()
                                                             for o in oms])
            h.sync()
            qg = [t.cpu().numpy() for t in res["Q"]]
            sub = [M.subspace(qg[n], ref["Q"][n]) for n in range(N)]
            e = float(res["err"][0])
            print(f"{name:4s} {vname:11s} subspace " + " ".join(f"{s:.2e}" for s in sub) +
                  f"  E rel {abs(e - ref['E']) / ref['E']:.2e}", flush=True)
            h.close()


if __name__ == "__main__":
    main()
