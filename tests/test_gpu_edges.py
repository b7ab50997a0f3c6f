"""Edge cases of the hot path on the GPU against the fp64 oracle: the order limits (N = 2, a
randomized SVD; N = 5), the maximum sketch width K_n = 128, the K_n > 128 and empty-mode
rejections."""
import dataclasses

import numpy as np
import pytest

import oracle
from gen import synth
from tests import _metrics as M

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2001_07124_b200 import api
    return api


@pytest.fixture(scope="module")
def h(P):
    hh = P.Handle()
    yield hh
    hh.close()


def _dev(x):
    return torch.from_numpy(synth.to_device_layout(x)).cuda()


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check(P, res, ref, tol=1e-5):
    qg = [q.cpu().numpy() for q in res["Q"]]
    gg = P.core_to_numpy(res["G"])
    for n, q in enumerate(qg):
        assert M.orth(q) <= 1e-12
        assert M.subspace(q, ref["Q"][n]) <= tol, (n, M.subspace(q, ref["Q"][n]))
    assert M.recon(gg, qg, ref["G"], ref["Q"]) <= tol
    assert abs(float(res["err"][0]) - ref["E"]) / ref["E"] <= tol


@pytest.mark.parametrize("q", [0, 1])
def test_order2_randomized_svd(P, h, q):
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"].scaled((300, 200), (12, 12), (12, 12)), q=q)
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(2)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=q)
    res = P.rtucker_hosvd(h, _dev(x), cfg.ranks, cfg.p, q, [_t(o) for o in oms])
    h.sync()
    _check(P, res, ref)


def test_order5_hosvd_and_sthosvd(P, h):
    cfg = dataclasses.replace(synth.CONFIGS["cfg3"].scaled((12, 11, 10, 9, 8), (3, 3, 3, 3, 3), (3, 3, 3, 3, 2)),
                              p=2, q=1)
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(5)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    res = P.rtucker_hosvd(h, _dev(x), cfg.ranks, cfg.p, 1, [_t(o) for o in oms])
    h.sync()
    _check(P, res, ref)
    rng = np.random.default_rng(71)
    st = []
    for n in range(5):
        d = synth.sthosvd_dims_before(cfg, n)
        J = int(np.prod(d)) // d[n]
        st.append(rng.standard_normal((J, min(cfg.ranks[n] + cfg.p, d[n], J))).astype(np.float32))
    ref2 = oracle.sthosvd(x, cfg.ranks, st, q=1)
    res2 = P.rtucker_sthosvd(h, _dev(x), cfg.ranks, cfg.p, 1, [_t(o) for o in st])
    h.sync()
    _check(P, res2, ref2)


def test_max_sketch_width_128(P, h):
    """K_n = R_n + p = 128, the widest tensor-core tile (NPAD = 128), with a power iteration."""
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled((256, 200, 160), (112, 112, 112), (112, 112, 112)),
                              p=16, q=1)
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    assert all(o.shape[1] == 128 for o in oms)
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    res = P.rtucker_hosvd(h, _dev(x), cfg.ranks, cfg.p, 1, [_t(o) for o in oms])
    h.sync()
    _check(P, res, ref)


def test_rejections(P, h):
    from paper_2001_07124_b200 import _lib as L
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled((256, 200, 160), (8, 8, 8), (113, 113, 113)), p=16)
    x = _dev(synth.make_tensor(dataclasses.replace(cfg, ranks=(8, 8, 8))))
    oms = [_t(np.zeros((cfg.J(n), 129), np.float32)) for n in range(3)]
    with pytest.raises(L.RtError) as e:                  # K_n = 129 > 128
        P.rtucker_hosvd(h, x, cfg.ranks, cfg.p, 0, oms)
    assert e.value.status == -7
    empty = torch.empty((0, 4, 4), dtype=torch.float32, device="cuda")
    with pytest.raises(L.RtError) as e:                  # a mode of size 0
        P.rtucker_sketch(h, empty, 0, _t(np.zeros((0, 2), np.float32)))
    assert e.value.status == -1
    h.sync()
