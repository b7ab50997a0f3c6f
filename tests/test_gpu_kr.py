"""GPU parity of the Khatri-Rao sketch (P:510 footnote, KR product P:317)
through the C-ABI (kind "kr") against the fp64 oracle on the same seeded inputs."""
import threading

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
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("dims,K,dtype", [
    ((37, 50, 29), 13, np.float32),          # ragged
    ((20, 18, 16, 14), 9, np.float32),       # order 4: one TTM + two TTV stages
    ((130, 7, 300), 6, np.float32),
    ((300, 260), 40, np.float32),            # order 2: the TTM stage only
    ((24, 22, 20), 11, np.float64),
])
def test_kr_sketch_parity(P, h, dims, K, dtype):
    rng = np.random.default_rng(31)
    x = np.asfortranarray(rng.standard_normal(dims).astype(dtype))
    X = _dev(x)
    tol = 1e-5 if dtype == np.float32 else 1e-12
    for n in range(len(dims)):
        k = min(K, dims[n], x.size // dims[n])
        oms = [None if j == n else rng.standard_normal((dims[j], k)).astype(dtype) for j in range(len(dims))]
        y = P.rtucker_sketch(h, X, n, [_t(o) for o in oms], kind="kr").cpu().numpy()
        y0, _ = oracle.sketch_kr(x, n, oms)
        assert M.rel_fro(y, y0) <= tol, (n, M.rel_fro(y, y0))
    h.sync()


@pytest.mark.parametrize("q", [0, 1])
def test_kr_hosvd_parity(P, h, q):
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"].scaled((120, 110, 100), (10, 10, 10), (10, 10, 10)), q=q)
    x = synth.make_tensor(cfg)
    oms = [synth.kr_omegas(cfg, n, cfg.dims) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=q, kind="kr")
    res = P.rtucker_hosvd(h, _dev(x), cfg.ranks, cfg.p, q, [[_t(o) for o in row] for row in oms], kind="kr")
    h.sync()
    qg = [t.cpu().numpy() for t in res["Q"]]
    gg = P.core_to_numpy(res["G"])
    for n in range(3):
        assert M.orth(qg[n]) <= 1e-12
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert M.core_in_oracle_basis(gg, qg, ref["G"], ref["Q"]) <= 1e-5
    assert M.recon(gg, qg, ref["G"], ref["Q"]) <= 1e-5
    assert abs(float(res["err"][0]) - ref["E"]) / ref["E"] <= 1e-5


def test_kr_sthosvd_parity(P, h):
    cfg = synth.CONFIGS["cfg3"].scaled((40, 36, 32, 30), (6, 6, 6, 6), (6, 6, 6, 6))
    x = synth.make_tensor(cfg)
    oms = [synth.kr_omegas(cfg, n, synth.sthosvd_dims_before(cfg, n)) for n in range(4)]
    ref = oracle.sthosvd(x, cfg.ranks, oms, q=0, kind="kr")
    res = P.rtucker_sthosvd(h, _dev(x), cfg.ranks, cfg.p, 0, [[_t(o) for o in row] for row in oms], kind="kr")
    h.sync()
    qg = [t.cpu().numpy() for t in res["Q"]]
    for n in range(4):
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert abs(float(res["err"][0]) - ref["E"]) / ref["E"] <= 1e-5


def test_kr_invalid_widths(P, h):
    from paper_2001_07124_b200 import _lib as L
    x = _dev(np.asfortranarray(np.ones((8, 9, 10), np.float32)))
    oms = [None, _t(np.ones((9, 3), np.float32)), _t(np.ones((10, 4), np.float32))]   # K mismatch
    with pytest.raises(L.RtError):
        P.rtucker_sketch(h, x, 0, oms, kind="kr")
    h.sync()


@pytest.mark.parametrize("nranks", [2])
def test_kr_loopback_multirank(P, nranks):
    """Slab-parallel KR sketches: for modes n < N-1 the last-mode factor holds the slab's rows and
    the TTV partial sums are allreduced (C1); the last mode's sketch rows stay local."""
    cfg = synth.CONFIGS["cfg5"].scaled((40, 36, 32), (5, 5, 5), (5, 5, 5))
    x = synth.make_tensor(cfg)
    oms = [synth.kr_omegas(cfg, n, cfg.dims) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=cfg.q, kind="kr")
    cuts = np.linspace(0, cfg.dims[2], nranks + 1).astype(int)
    grp = P.LoopbackGroup(nranks)
    out, errs = [None] * nranks, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                hh = P.Handle(stream=s, loopback_group=grp, rank=r)
                lo, hi = int(cuts[r]), int(cuts[r + 1])
                xs = _dev(np.asfortranarray(x[:, :, lo:hi]))
                loc = [[None if o is None else _t(o[lo:hi] if k == 2 else o) for k, o in enumerate(row)]
                       for row in oms]
                res = P.rtucker_hosvd(hh, xs, cfg.ranks, cfg.p, cfg.q, loc, kind="kr", last_offset=lo,
                                      last_global=cfg.dims[2])
                hh.sync()
                out[r] = dict(Q=[t.cpu().numpy() for t in res["Q"]], G=P.core_to_numpy(res["G"]),
                              err=res["err"].cpu().numpy())
                hh.close()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    qg = out[0]["Q"][:2] + [np.concatenate([out[r]["Q"][2] for r in range(nranks)], axis=0)]
    for n in range(3):
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert abs(out[0]["err"][0] - ref["E"]) / ref["E"] <= 1e-5


@pytest.mark.parametrize("dims,K", [((128, 96, 64), 40), ((256, 36, 20, 12), 16), ((40, 36, 32), 13)])
def test_kr_sketch_tf32_exact_factors(P, dims, K):
    """RT_OPT_OMEGA_TF32 with host-rounded Khatri-Rao factors: the first TTM runs 2 tensor products
    (no B split) and still matches the oracle on the same rounded factors."""
    from paper_2001_07124_b200 import _lib as L
    rng = np.random.default_rng(35)
    x = np.asfortranarray(rng.standard_normal(dims).astype(np.float32))
    hh = P.Handle()
    hh.set_option(L.RT_OPT_OMEGA_TF32, 1)
    X = _dev(x)
    for n in range(len(dims)):
        k = min(K, dims[n], x.size // dims[n])
        oms = [None if j == n else synth.round_tf32(rng.standard_normal((dims[j], k))) for j in range(len(dims))]
        y = P.rtucker_sketch(hh, X, n, [_t(o) for o in oms], kind="kr").cpu().numpy()
        y0, _ = oracle.sketch_kr(x, n, oms)
        assert M.rel_fro(y, y0) <= 1e-5, (n, M.rel_fro(y, y0))
    hh.sync()
    hh.close()
