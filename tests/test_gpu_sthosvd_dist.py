"""Slab-parallel R-STHOSVD (Alg.8: "STHOSVD in ascending order also shards
cleanly") on one GPU through the loopback communicator, against the fp64 oracle on the whole tensor.
Modes 0..N-2 shrink the local slab (their sketches and the Grams of B_(n) are slab partial sums);
the slab mode comes last (local sketch rows, TSQR, B allreduced, local factor rows)."""
import math
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


def _t(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _gauss_sthosvd_omegas(cfg, seed):
    """Gaussian Omega of each step, sized for the shrinking working tensor (rows in the j order)."""
    rng = np.random.default_rng(seed)
    out = []
    for n in range(cfg.order):
        d = synth.sthosvd_dims_before(cfg, n)
        J = math.prod(d) // d[n]
        K = min(cfg.ranks[n] + cfg.p, d[n], J)
        out.append(rng.standard_normal((J, K)).astype(cfg.np_dtype))
    return out


def _run(P, x, cfg, nranks, kind, oms, q):
    N = cfg.order
    cuts = np.linspace(0, cfg.dims[-1], nranks + 1).astype(int)
    grp = P.LoopbackGroup(nranks)
    out, errs = [None] * nranks, []

    def local_omegas(lo, hi):
        loc = []
        for n in range(N):
            d = synth.sthosvd_dims_before(cfg, n)
            if kind == "gauss":
                if n == N - 1:
                    loc.append(_t(oms[n]))
                else:
                    a = math.prod(d[k] for k in range(N - 1) if k != n)     # j = alpha + a * i_last
                    loc.append(_t(oms[n][a * lo:a * hi]))
            else:
                loc.append([None if o is None else _t(o[lo:hi] if k == N - 1 else o) for k, o in enumerate(oms[n])])
        return loc

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                hh = P.Handle(stream=s, loopback_group=grp, rank=r)
                lo, hi = int(cuts[r]), int(cuts[r + 1])
                xs = torch.from_numpy(synth.to_device_layout(np.asfortranarray(x[..., lo:hi]))).cuda()
                res = P.rtucker_sthosvd(hh, xs, cfg.ranks, cfg.p, q, local_omegas(lo, hi), kind=kind,
                                        last_offset=lo, last_global=cfg.dims[-1])
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
    qg = out[0]["Q"][:N - 1] + [np.concatenate([out[r]["Q"][N - 1] for r in range(nranks)], axis=0)]
    return qg, out


@pytest.mark.parametrize("nranks", [2, 3])
@pytest.mark.parametrize("q", [0, 1])
def test_sthosvd_gauss_loopback(P, nranks, q):
    cfg = synth.CONFIGS["cfg3"].scaled((40, 36, 32, 30), (6, 6, 6, 6), (6, 6, 6, 6))
    x = synth.make_tensor(cfg)
    oms = _gauss_sthosvd_omegas(cfg, 61 + q)
    ref = oracle.sthosvd(x, cfg.ranks, oms, q=q)
    qg, out = _run(P, x, cfg, nranks, "gauss", oms, q)
    for n in range(cfg.order):
        assert M.orth(qg[n]) <= 1e-12
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5, (n, M.subspace(qg[n], ref["Q"][n]))
    assert M.recon(out[0]["G"], qg, ref["G"], ref["Q"]) <= 1e-5
    for r in range(nranks):
        assert abs(out[r]["err"][0] - ref["E"]) / ref["E"] <= 1e-5


def test_sthosvd_kron_loopback(P):
    cfg = synth.CONFIGS["cfg3"].scaled((40, 36, 32, 30), (6, 6, 6, 6), (6, 6, 6, 6))
    x = synth.make_tensor(cfg)
    oms = [synth.kron_omegas(cfg, n, synth.sthosvd_dims_before(cfg, n)) for n in range(4)]
    ref = oracle.sthosvd(x, cfg.ranks, oms, q=0, kind="kron")
    qg, out = _run(P, x, cfg, 2, "kron", oms, 0)
    for n in range(cfg.order):
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert abs(out[0]["err"][0] - ref["E"]) / ref["E"] <= 1e-5


def test_sthosvd_sharded_needs_slab_mode_last(P):
    from paper_2001_07124_b200 import _lib as L
    cfg = synth.CONFIGS["cfg3"].scaled((20, 18, 16, 14), (4, 4, 4, 4), (4, 4, 4, 4))
    x = synth.make_tensor(cfg)
    grp = P.LoopbackGroup(1)
    hh = P.Handle(loopback_group=grp, rank=0)
    xs = torch.from_numpy(synth.to_device_layout(np.asfortranarray(x[..., 0:7]))).cuda()
    oms = [[None] * 4 for _ in range(4)]
    with pytest.raises(L.RtError):
        P.rtucker_sthosvd(hh, xs, cfg.ranks, cfg.p, 0, oms, kind="kron", mode_order=[3, 2, 1, 0],
                          last_offset=0, last_global=14)
    hh.close()
