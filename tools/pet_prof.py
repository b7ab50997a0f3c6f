import torch, sys
sys.path.insert(0, "/root/repo")
from gen import synth
from paper_2001_07124_b200 import api
cfg = synth.CONFIGS["cfg5"]
h = api.Handle()
X, _ = synth.make_tensor_device(cfg, "cuda")
ks, ss = synth.pet_sizes(cfg)
om = [torch.from_numpy(synth.gaussian_omega(cfg, n, K=ks[n])).cuda() for n in range(3)]
omt = [torch.from_numpy(synth.omega_tilde(cfg, n, ss[n])).cuda() for n in range(3)]
api.rtucker_pet(h, X, cfg.ranks, om, omt); h.sync()
h.profile_read(); h.set_option(1, 1)
api.rtucker_pet(h, X, cfg.ranks, om, omt); h.sync()
prof, n = h.profile_read()
for nm, c, t in sorted(prof, key=lambda e: -e[2])[:15]: print(f"{nm:24s} {c:4d} {t:8.2f} ms")
