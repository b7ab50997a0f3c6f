"""One cfg3 R-STHOSVD call (Kronecker sketch, BASELINE configs[2]) after a warm-up call, for ncu
captures of the a2 (Kronecker chain) and a7 (STHOSVD shrink) kernels:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \\
        --log-file gpurun_out/cfg3.csv python tools/sthosvd_once.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from gen import synth
from paper_2001_07124_b200 import api as P

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
x = synth.make_tensor(cfg)
X = torch.from_numpy(synth.to_device_layout(x)).cuda()
ko = [[None if o is None else torch.from_numpy(np.ascontiguousarray(synth.round_tf32(o))).cuda()
       for o in synth.kron_omegas(cfg, n, synth.sthosvd_dims_before(cfg, n))] for n in range(cfg.order)]
h = P.Handle()
h.set_option(3, 1)
for _ in range(2):
    r = P.rtucker_sthosvd(h, X, cfg.ranks, cfg.p, cfg.q, ko, kind="kron")
    h.sync()
print("E =", float(r["err"][0]))
h.close()
