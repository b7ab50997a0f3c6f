"""Timeline of one cfg5 HOSVD step (or one rank's share of it): every library launch with its start
and end on the device, main and side streams together (RT_TIMELINE dump of rt_profile_read).  Shows
what is exposed on the critical path: gaps of the X-pass stream, the tail after the residual.

    python tools/timeline.py [--config cfg5] [--ranks 1] [--opt 0] [--min-us 20]
"""
import argparse
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--ranks", type=int, default=1, help="time rank 0's slab of a --ranks job (1-rank NCCL, forced collectives)")
ap.add_argument("--opt", type=int, default=0)
ap.add_argument("--min-us", type=float, default=20.0)
ap.add_argument("--algo", default="hosvd")
a = ap.parse_args()
path = tempfile.mktemp(suffix=".tl")
os.environ["RT_TIMELINE"] = path

import torch

from gen import synth
from paper_2001_07124_b200 import _lib as L
from paper_2001_07124_b200 import api as P
from paper_2001_07124_b200 import partition

cfg = synth.CONFIGS[a.config]
N = cfg.order
I_last = cfg.dims[-1]
lo, hi = partition.slab_range(I_last, a.ranks, 0)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    X, _ = synth.make_tensor_device(cfg, dev, last_range=(lo, hi))
    oms = []
    for n in range(N):
        r = partition.omega_rows(cfg.dims, n, lo, hi)
        if r is not None:
            oms.append(synth.gaussian_omega_device(cfg, n, dev, row0=r[0], rows=r[1], tf32=True))
        else:
            oms.append(synth.gaussian_omega_device(cfg, n, dev, tf32=True))
    if a.ranks > 1:
        h = P.Handle(stream=stream, nccl_id=P.get_unique_id(), nranks=1, rank=0)
        h.set_option(L.RT_OPT_FORCE_COLLECTIVES, 1)
    else:
        h = P.Handle(stream=stream)
    h.set_option(L.RT_OPT_OMEGA_TF32, 1)
    if a.opt:
        h.set_option(100, a.opt)

    def step():
        return P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms, last_offset=lo, last_global=I_last)

    for _ in range(3):
        step()
    h.sync()
    h.profile_read()
    if os.path.exists(path):
        os.remove(path)
    h.set_option(L.RT_OPT_PROFILE, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step()
    e1.record(stream)
    h.sync()
    h.set_option(L.RT_OPT_PROFILE, 0)
    h.profile_read()
print(f"step {e0.elapsed_time(e1):.3f} ms (profiling events on)")
rows = []
for line in open(path):
    if line.startswith("#"):
        continue
    nm, t0, t1 = line.split()
    rows.append((float(t0), float(t1), nm))
rows.sort()
end = 0.0
print(f"{'start':>9} {'end':>9} {'dur':>8}  name   (kernels under {a.min_us:.0f} us folded)")
small = {}
for t0, t1, nm in rows:
    end = max(end, t1)
    if (t1 - t0) * 1e3 < a.min_us:
        c = small.setdefault(nm, [0, 0.0])
        c[0] += 1
        c[1] += t1 - t0
        continue
    print(f"{t0:9.3f} {t1:9.3f} {t1 - t0:8.3f}  {nm}")
print(f"last launch ends at {end:.3f} ms")
print("folded:", ", ".join(f"{k} x{v[0]} {v[1] * 1e3:.0f}us" for k, v in sorted(small.items(), key=lambda kv: -kv[1][1])))
os.remove(path)
