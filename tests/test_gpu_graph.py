"""the C-ABI calls are stream-ordered and enqueue-only (no host synchronization in
the call), so a warmed-up rtucker_hosvd can be captured in a CUDA graph and replayed: the replay
reproduces the direct call exactly (same kernels, same order, same workspace)."""
import numpy as np
import pytest

from gen import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2001_07124_b200 import api
    return api


def test_hosvd_cuda_graph_replay(P):
    cfg = synth.CONFIGS["cfg2"].scaled((128, 120, 112), (10, 10, 10), (10, 10, 10))
    x = torch.from_numpy(synth.to_device_layout(synth.make_tensor(cfg))).cuda()
    oms = [torch.from_numpy(synth.gaussian_omega(cfg, n)).cuda() for n in range(3)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        h = P.Handle(stream=s)
        ref = P.rtucker_hosvd(h, x, cfg.ranks, cfg.p, cfg.q, oms)          # warm-up: workspace grown
        h.sync()
        ref_q = [q.clone() for q in ref["Q"]]
        ref_g, ref_e = ref["G"].clone(), ref["err"].clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            out = P.rtucker_hosvd(h, x, cfg.ranks, cfg.p, cfg.q, oms)
        for _ in range(2):
            g.replay()
        s.synchronize()
        for a, b in zip(out["Q"], ref_q):
            assert torch.equal(a, b)
        assert torch.equal(out["G"], ref_g)
        assert torch.equal(out["err"], ref_e)
        h.close()
