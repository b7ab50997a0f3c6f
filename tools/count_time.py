"""Time the count-sketch operator per mode on a device-generated BASELINE config (CUDA events)."""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from gen import synth
from paper_2001_07124_b200 import api

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg5")
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
h = api.Handle()
X, _ = synth.make_tensor_device(cfg, "cuda")
nbytes = X.numel() * X.element_size()
for n in range(cfg.order):
    codes, K = synth.count_codes(cfg, n)
    c = torch.from_numpy(codes).cuda()
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        y = api.rtucker_sketch(h, X, n, (c, K), kind="count")
        e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{a.cfg} mode {n} K={K} ms={ms:.2f} GB/s={nbytes / ms / 1e6:.0f}")
