"""Time RP-HOOI sweeps on a device-generated BASELINE config (default cfg5) with CUDA events."""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import synth
from paper_2001_07124_b200 import api

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg5")
ap.add_argument("--sweeps", type=int, default=1)
ap.add_argument("--ablate", type=int, default=0, help="RT_OPT_TC_ABLATE switch (220/221: S-chain X pass on TC off/on)")
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
h = api.Handle()
if a.ablate:
    h.set_option(100, a.ablate)
X = synth.make_tensor_device(cfg, "cuda")
if isinstance(X, tuple):
    X = X[0]
q0 = [torch.linalg.qr(torch.randn(d, r, dtype=torch.float64, device="cuda"))[0] for d, r in zip(cfg.dims, cfg.ranks)]
hs = [[torch.from_numpy(o).cuda() for o in sw] for sw in synth.hooi_omegas(cfg, a.sweeps)]
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(h.stream)
    res = api.rtucker_rp_hooi(h, X, cfg.ranks, q0, hs)
    e1.record(h.stream); torch.cuda.synchronize()
    print(f"{a.cfg} sweeps={a.sweeps} ms={e0.elapsed_time(e1):.1f} E={float(res['err'][0]):.6g}")
