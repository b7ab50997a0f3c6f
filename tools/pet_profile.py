"""Per-label device times of one cfg5 R-PET call (bench_rows.py's inputs), from the library's events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from gen import synth
from paper_2001_07124_b200 import _lib as L
from paper_2001_07124_b200 import api

cfg = synth.CONFIGS["cfg5"]
N = cfg.order
X, _ = synth.make_tensor_device(cfg, "cuda")
h = api.Handle()
h.set_option(L.RT_OPT_OMEGA_TF32, 1)
ks, ss = synth.pet_sizes(cfg)
om = [torch.from_numpy(synth.round_tf32(synth.gaussian_omega(cfg, n, K=ks[n]))).cuda() for n in range(N)]
omt = [torch.from_numpy(synth.round_tf32(synth.omega_tilde(cfg, n, ss[n]))).cuda() for n in range(N)]
print("K", ks, "S", ss)
api.rtucker_pet(h, X, cfg.ranks, om, omt)
h.sync()
h.profile_read()
h.set_option(L.RT_OPT_PROFILE, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
api.rtucker_pet(h, X, cfg.ranks, om, omt)
e1.record()
h.sync()
torch.cuda.synchronize()
print("call ms", e0.elapsed_time(e1))
for n, c, ms in sorted(h.profile_read()[0], key=lambda e: -e[2])[:20]:
    print(f"  {n:24s} {c:4d}x {ms:8.3f} ms")
