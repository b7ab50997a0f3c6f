"""HOSVD step of one BASELINE config (default cfg5): direct C-ABI calls vs replay of a CUDA graph captured
from the same call.   python tools/graph_time.py [cfg2]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from gen import synth
from paper_2001_07124_b200 import api as P

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5"]
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    X, _ = synth.make_tensor_device(cfg, "cuda")
    oms = [synth.gaussian_omega_device(cfg, n, "cuda", tf32=True) for n in range(3)]
    torch.cuda.synchronize()
    h = P.Handle(stream=s)
    h.set_option(3, 1)
    step = lambda: P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms)
    for _ in range(3):
        step()
    h.sync()
    def timed(fn, k=20 if cfg.nbytes < (1 << 33) else 5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(s)
        for _ in range(k):
            fn()
        e1.record(s); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / k
    print("direct ms/step", timed(step))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    g.replay(); torch.cuda.synchronize()
    print("graph  ms/step", timed(g.replay))
    print("direct ms/step", timed(step))
