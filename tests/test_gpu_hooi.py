"""GPU parity of RP-HOOI (Alg.7) through the C-ABI
(`rtucker_rp_hooi`) against the fp64 oracle `oracle.rp_hooi` on the same seeded inputs (the same
starting factors, the oracle's RP-HOSVD output, and the same per-sweep Omega^(n)).  Metrics and
tolerances as for the HOSVD path (M2, M4, M5 <= 1e-5; orthonormality <= 1e-12).  E: the default
path streams X on the tensor cores (fp32-accurate), so E is held to DESIGN.md reading R30,
|E_gpu - E_o| <= max(1e-5 E_o, 4u) with u = 2^-24; the fp64 X pass (RT_OPT_TC_ABLATE 220, reading
R25) is held to the plain relative 1e-5 bar on the same cases."""
import dataclasses
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


@pytest.fixture(scope="module")
def h64(P):
    hh = P.Handle()
    hh.set_option(100, 220)                 # RT_OPT_TC_ABLATE 220: fp64 X pass of the S chains (R25)
    yield hh
    hh.close()


U32 = 2.0 ** -24


def _e_ok(e, e_ref, strict):
    """R30 (tensor-core X pass): max(1e-5 E, 4u) absolute floor; R25 (fp64 X pass): relative 1e-5."""
    return abs(e - e_ref) <= (1e-5 * e_ref if strict else max(1e-5 * e_ref, 4 * U32))


def _dev(x):
    return torch.from_numpy(synth.to_device_layout(x)).cuda()


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _start(cfg, x):
    oms = [synth.gaussian_omega(cfg, n) for n in range(cfg.order)]
    return oracle.hosvd(x, cfg.ranks, oms, q=0)["Q"]


def _check(P, res, ref, tol=1e-5, strict=False):
    qg = [q.cpu().numpy() for q in res["Q"]]
    gg = P.core_to_numpy(res["G"])
    for n, q in enumerate(qg):
        assert M.orth(q) <= 1e-12
        assert M.subspace(q, ref["Q"][n]) <= tol, ("M2", n, M.subspace(q, ref["Q"][n]))
    assert M.core_in_oracle_basis(gg, qg, ref["G"], ref["Q"]) <= tol
    assert M.recon(gg, qg, ref["G"], ref["Q"]) <= tol
    e = float(res["err"][0])
    assert _e_ok(e, ref["E"], strict), (e, ref["E"], abs(e - ref["E"]) / ref["E"])


CASES = {
    "cfg2s": (synth.CONFIGS["cfg2"].scaled((150, 140, 130), (12, 12, 12), (12, 12, 12)), 2),
    "cfg5s": (synth.CONFIGS["cfg5"].scaled((160, 150, 140), (24, 24, 24), (24, 24, 24)), 1),
    "cfg4s": (synth.CONFIGS["cfg4"].scaled((300, 280, 64), (100, 100, 50), (30, 30, 12)), 2),
    "order4": (synth.CONFIGS["cfg3"].scaled((40, 36, 32, 30), (6, 6, 6, 6), (6, 5, 4, 6)), 2),
    "ragged": (synth.CONFIGS["cfg2"].scaled((37, 50, 29), (5, 5, 5), (5, 3, 4)), 3),
    "f64": (synth.CONFIGS["cfg1"].scaled((40, 36, 32), (5, 5, 5), (5, 5, 5)), 2),
}


@pytest.mark.parametrize("strict", [False, True])
@pytest.mark.parametrize("name", list(CASES))
def test_rp_hooi_parity(P, h, h64, name, strict):
    cfg, sweeps = CASES[name]
    x = synth.make_tensor(cfg)
    q0 = _start(cfg, x)
    oms = synth.hooi_omegas(cfg, sweeps)
    ref = oracle.rp_hooi(x, cfg.ranks, q0, oms)
    hh = h64 if strict else h
    res = P.rtucker_rp_hooi(hh, _dev(x), cfg.ranks, [_t(q) for q in q0], [[_t(o) for o in s] for s in oms])
    hh.sync()
    _check(P, res, ref, strict=strict)


@pytest.mark.parametrize("strict", [False, True])
def test_rp_hooi_gaussian_start(P, h, h64, strict):
    """Alg.7 line 1 allows a random start: unnormalized Gaussian Q_init (entries |q| >= 4 occur,
    outside the fp16 split's range once scaled by 2^14).  The fp16-split X pass is gated on the
    device by max|Q| < 2 as well as X's scale, so the wide start factors send sweep 0's first
    stages to the 3xTF32 twin (the run counters show both kinds ran); parity with the oracle from
    the same start."""
    # dims multiples of 4: the first S-chain stage takes the tensor-core path (16-byte TMA strides)
    cfg = synth.CONFIGS["cfg2"].scaled((152, 144, 128), (12, 12, 12), (12, 12, 12))
    x = synth.make_tensor(cfg)
    q0 = [synth.rng_for(4242, 7, n).standard_normal((cfg.dims[n], cfg.ranks[n])) * 3.0 for n in range(3)]
    assert max(np.abs(q).max() for q in q0) >= 4.0
    oms = synth.hooi_omegas(cfg, 2)
    ref = oracle.rp_hooi(x, cfg.ranks, q0, oms)
    hh = h64 if strict else h
    hh.profile_read()
    res = P.rtucker_rp_hooi(hh, _dev(x), cfg.ranks, [_t(q) for q in q0], [[_t(o) for o in s] for s in oms])
    hh.sync()
    runs = {n: c for n, c, _ in hh.profile_read()[0] if n in ("h16_ran", "tf32_twin_ran")}
    if not strict:
        assert runs.get("tf32_twin_ran", 0) >= 1 and runs.get("h16_ran", 0) >= 1, runs
    assert all(np.isfinite(q.cpu().numpy()).all() for q in res["Q"])
    _check(P, res, ref, strict=strict)


def test_rp_hooi_zero_sweeps_is_core_of_start(P, h):
    """sweeps = 0: the factors are the (sign-canonicalized) starting factors and G their core."""
    cfg = synth.CONFIGS["cfg2"].scaled((60, 50, 40), (5, 5, 5), (5, 5, 5))
    x = synth.make_tensor(cfg)
    q0 = _start(cfg, x)
    ref = oracle.rp_hooi(x, cfg.ranks, q0, [])
    res = P.rtucker_rp_hooi(h, _dev(x), cfg.ranks, [_t(q) for q in q0], [])
    h.sync()
    _check(P, res, ref)


def test_rp_hooi_exact_rank_fp64(P, h):
    """Exact multilinear rank (no noise), fp64: a sweep from the RP-HOSVD start keeps E < 1e-10."""
    cfg = dataclasses.replace(synth.CONFIGS["cfg1"].scaled((40, 36, 32), (4, 4, 4), (4, 4, 4)), noise="none")
    x = synth.make_tensor(cfg)
    q0 = _start(cfg, x)
    res = P.rtucker_rp_hooi(h, _dev(x), cfg.ranks, [_t(q) for q in q0], [[_t(o) for o in s]
                                                                        for s in synth.hooi_omegas(cfg, 1)])
    h.sync()
    assert float(res["err"][0]) < 1e-10


def test_rp_hooi_not_worse_than_hooi_bound(P, h):
    """E_rphooi >= E_hooi (1 - 1e-6) (pin P27 on the GPU result, tf32-free fp32 data path)."""
    cfg = synth.CONFIGS["cfg2"].scaled((24, 22, 20), (4, 4, 4), (4, 4, 4))
    x = synth.make_tensor(cfg)
    q0 = _start(cfg, x)
    res = P.rtucker_rp_hooi(h, _dev(x), cfg.ranks, [_t(q) for q in q0], [[_t(o) for o in s]
                                                                        for s in synth.hooi_omegas(cfg, 3)])
    h.sync()
    assert oracle.hooi(x, cfg.ranks)["E"] * (1 - 1e-6) <= float(res["err"][0])


def test_rp_hooi_invalid_arguments(P, h):
    from paper_2001_07124_b200 import _lib as L
    cfg = synth.CONFIGS["cfg2"].scaled((37, 50, 29), (5, 5, 5), (5, 5, 5))
    x = synth.make_tensor(cfg)
    q0 = _start(cfg, x)
    oms = synth.hooi_omegas(cfg, 1)
    bad = [[_t(o[:, :-1]) for o in s] for s in oms]                       # Omega width R_n - 1
    with pytest.raises(ValueError):
        P.rtucker_rp_hooi(h, _dev(x), cfg.ranks, [_t(q) for q in q0], bad)
    big = (5, 5, 30)                                                       # R_3 > I_3
    with pytest.raises(L.RtError):
        P.rtucker_rp_hooi(h, _dev(x), big, [_t(q) for q in q0], [])
    h.sync()


@pytest.mark.parametrize("strict", [False, True])
@pytest.mark.parametrize("nranks", [2, 3])
def test_rp_hooi_loopback_multirank(P, nranks, strict):
    """Slab-parallel RP-HOOI on one GPU (loopback communicator): S for n < N-1 contracts the
    distributed last mode (allreduced partial sums); Q^(N-1) is row-distributed (TSQR gather)."""
    cfg = synth.CONFIGS["cfg5"].scaled((48, 40, 36), (6, 6, 6), (6, 6, 6))
    x = synth.make_tensor(cfg)
    q0 = _start(cfg, x)
    oms = synth.hooi_omegas(cfg, 2)
    ref = oracle.rp_hooi(x, cfg.ranks, q0, oms)
    cuts = np.linspace(0, cfg.dims[2], nranks + 1).astype(int)
    grp = P.LoopbackGroup(nranks)
    out = [None] * nranks
    errs = []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                hh = P.Handle(stream=s, loopback_group=grp, rank=r)
                if strict:
                    hh.set_option(100, 220)
                lo, hi = int(cuts[r]), int(cuts[r + 1])
                xs = _dev(np.asfortranarray(x[:, :, lo:hi]))
                ql = [_t(q0[0]), _t(q0[1]), _t(q0[2][lo:hi])]
                res = P.rtucker_rp_hooi(hh, xs, cfg.ranks, ql, [[_t(o) for o in sw] for sw in oms],
                                        last_offset=lo, last_global=cfg.dims[2])
                hh.sync()
                out[r] = dict(Q=[q.cpu().numpy() for q in res["Q"]], G=P.core_to_numpy(res["G"]),
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
    q_last = np.concatenate([out[r]["Q"][2] for r in range(nranks)], axis=0)
    qg = out[0]["Q"][:2] + [q_last]
    for n in range(3):
        assert M.orth(qg[n]) <= 1e-12
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert M.recon(out[0]["G"], qg, ref["G"], ref["Q"]) <= 1e-5
    assert _e_ok(out[0]["err"][0], ref["E"], strict), (out[0]["err"][0], ref["E"])
