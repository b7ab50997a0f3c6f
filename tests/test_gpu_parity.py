"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 oracle on the same seeded
inputs.  Tolerances (BASELINE.json north_star): relative Frobenius <= 1e-5 on sketches
and cores, |E_gpu - E_oracle| / E_oracle <= 1e-5; orthonormality <= 1e-12 (fp64 QR/EVD).
"""
import dataclasses
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
    import paper_2001_07124_b200 as pkg
    from paper_2001_07124_b200 import api
    return api


@pytest.fixture(scope="module")
def h(P):
    hh = P.Handle()
    yield hh
    hh.close()


def dev(x_np, dtype=None):
    t = torch.from_numpy(synth.to_device_layout(x_np if dtype is None else x_np.astype(dtype)))
    return t.cuda()


def mat(t):
    return t.detach().cpu().numpy()


def om_dev(om):
    return torch.from_numpy(np.ascontiguousarray(om)).cuda()


def rand_tensor(seed, dims, dtype=np.float32):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal(dims).astype(dtype))


# --------------------------------------------------------------------- sketch (a1)
@pytest.mark.parametrize("dims,K,dtype", [
    ((37, 50, 29), 13, np.float32),          # ragged tails in every mode
    ((130, 7, 300), 30, np.float32),         # several i-tiles, tiny middle mode
    ((9, 17, 5, 33), 24, np.float32),        # order 4
    ((300, 260), 80, np.float32),            # order 2, K = 80
    ((3, 4, 5, 6, 7), 5, np.float32),        # order 5
    ((40, 33, 21), 10, np.float64),          # fp64 path
])
def test_sketch_gauss_parity(P, h, dims, K, dtype):
    x = rand_tensor(1, dims, dtype)
    X = dev(x)
    rng = np.random.default_rng(2)
    tol = 1e-5 if dtype == np.float32 else 1e-12
    for n in range(len(dims)):
        J = x.size // dims[n]
        k = min(K, dims[n], J)
        om = rng.standard_normal((J, k)).astype(dtype)
        y = mat(P.rtucker_sketch(h, X, n, om_dev(om)))
        y0, _ = oracle.sketch_gauss(x, n, om, 0)
        assert M.rel_fro(y, y0) <= tol, (n, M.rel_fro(y, y0))
    h.sync()


@pytest.mark.parametrize("q", [1, 2])
def test_sketch_power_iteration_subspace(P, h, q):
    """a3: the power-iterated sketch spans the oracle's subspace (R2 reading)."""
    cfg = synth.CONFIGS["cfg2"].scaled((60, 50, 40), (6, 6, 6), (6, 6, 6))
    x = synth.make_tensor(cfg)
    X = dev(x)
    for n in range(3):
        om = synth.gaussian_omega(cfg, n, K=10)
        y = mat(P.rtucker_sketch(h, X, n, om_dev(om), q=q))
        _, yo = oracle.sketch_gauss(x, n, om, q)
        qg, _ = np.linalg.qr(y)
        qo, _ = np.linalg.qr(yo)
        # top-6 (signal) directions agree; compare the dominant subspace of the sketches
        ug = np.linalg.svd(y, full_matrices=False)[0][:, :6]
        uo = np.linalg.svd(yo, full_matrices=False)[0][:, :6]
        assert M.subspace(ug, uo) <= 1e-5
        assert M.subspace(qg, qo) <= 1e-3     # whole K-dim span incl. noise directions
    h.sync()


def test_sketch_kron_parity(P, h):
    """a2: Kronecker sketch = X_(n)(Omega_N kron ... kron Omega_1) (Eq.(2))."""
    dims = (20, 18, 16, 14)
    x = rand_tensor(3, dims)
    X = dev(x)
    rng = np.random.default_rng(4)
    for n in range(4):
        oms = [None if k == n else rng.standard_normal((dims[k], 2 + (k % 2))).astype(np.float32) for k in range(4)]
        y = mat(P.rtucker_sketch(h, X, n, [None if o is None else om_dev(o) for o in oms], kind="kron"))
        y0, _ = oracle.sketch_kron(x, n, oms, 0)
        assert M.rel_fro(y, y0) <= 1e-5
    h.sync()


# ------------------------------------------------------------------------ QR (a4)
@pytest.mark.parametrize("m,k,cond", [(500, 30, 1.0), (2048, 80, 1e4), (777, 13, 1e8), (64, 64, 10.0), (5, 1, 1.0)])
def test_qr_parity(P, h, m, k, cond):
    rng = np.random.default_rng(5)
    u, _ = np.linalg.qr(rng.standard_normal((m, k)))
    v, _ = np.linalg.qr(rng.standard_normal((k, k)))
    s = np.logspace(0, -math.log10(cond), k) if cond > 1 else np.ones(k)
    y = (u * s) @ v.T
    Q, R = P.rtucker_qr(h, torch.from_numpy(y).cuda())
    h.sync()
    q, r = mat(Q), mat(R)
    qo, ro = oracle.qr_plus(y)
    assert M.orth(q) <= 1e-12
    assert np.all(np.diag(r) >= 0)
    assert M.rel_fro(q @ r, y) <= 1e-12
    assert M.rel_fro(q, qo) <= 1e-14 * cond + 1e-12


def test_qr_fp32_input_and_zero(P, h):
    y = np.random.default_rng(6).standard_normal((300, 20)).astype(np.float32)
    Q, R = P.rtucker_qr(h, torch.from_numpy(y).cuda())
    h.sync()
    qo, ro = oracle.qr_plus(y.astype(np.float64))
    assert M.rel_fro(mat(Q), qo) <= 1e-12
    Q0, R0 = P.rtucker_qr(h, torch.zeros((50, 7), dtype=torch.float64).cuda())
    h.sync()
    np.testing.assert_array_equal(mat(Q0), np.eye(50, 7))
    np.testing.assert_array_equal(mat(R0), np.zeros((7, 7)))


# ---------------------------------------------------------------------- core (a5)
@pytest.mark.parametrize("dims,C,dtype", [((37, 50, 29), (5, 7, 3), np.float32),
                                          ((20, 30, 10, 12), (4, 5, 6, 7), np.float32),
                                          ((40, 33, 21), (6, 6, 6), np.float64)])
def test_core_and_error_parity(P, h, dims, C, dtype):
    x = rand_tensor(7, dims, dtype)
    rng = np.random.default_rng(8)
    qs = [np.linalg.qr(rng.standard_normal((d, c)))[0] for d, c in zip(dims, C)]
    G, err = P.rtucker_core(h, dev(x), [torch.from_numpy(q).cuda() for q in qs])
    h.sync()
    g = P.core_to_numpy(G)
    go = oracle.core(x, qs)
    tol = 1e-5 if dtype == np.float32 else 1e-12
    assert M.rel_fro(g, go) <= tol
    e = mat(err)
    eo = oracle.rel_error(x, go, qs)
    assert abs(e[0] - eo) / eo <= tol
    assert abs(e[1] - oracle.rel_error_gram(x, go)) <= 1e-6


# --------------------------------------------------------- end to end (a1-a8)
def _omegas_for(cfg, kind="gauss", sthosvd=False):
    N = cfg.order
    if kind == "gauss":
        if not sthosvd:
            return [synth.gaussian_omega(cfg, n) for n in range(N)]
        oms = []
        d = list(cfg.dims)
        for n in range(N):
            J = int(np.prod([d[k] for k in range(N) if k != n]))
            K = min(cfg.ranks[n] + cfg.p, d[n], J)
            oms.append(np.ascontiguousarray(
                synth.rng_for(cfg.cfg_id, 40, n).standard_normal((J, K)).astype(cfg.np_dtype)))
            d[n] = cfg.ranks[n]
        return oms
    if sthosvd:
        return [synth.kron_omegas(cfg, n, synth.sthosvd_dims_before(cfg, n)) for n in range(N)]
    return [synth.kron_omegas(cfg, n, cfg.dims) for n in range(N)]


def _to_dev_omegas(oms, kind):
    if kind == "gauss":
        return [om_dev(o) for o in oms]
    return [[None if o is None else om_dev(o) for o in row] for row in oms]


def _check_result(res, ref, cfg, tol=1e-5, sketch_tol=1e-5):
    qg = [mat(q) for q in res["Q"]]
    gg = P_core(res["G"])
    e = mat(res["err"])
    for n, q in enumerate(qg):
        assert M.orth(q) <= 1e-12, ("M7", n, M.orth(q))
        assert M.subspace(q, ref["Q"][n]) <= tol, ("M2", n, M.subspace(q, ref["Q"][n]))
    assert M.core_in_oracle_basis(gg, qg, ref["G"], ref["Q"]) <= tol
    assert M.recon(gg, qg, ref["G"], ref["Q"]) <= tol
    if ref["E"] > 1e-12:
        assert abs(e[0] - ref["E"]) / ref["E"] <= tol, ("M6", e[0], ref["E"])
    else:
        assert abs(e[0]) <= 1e-6
    return qg, gg, e


def P_core(G):
    return G.detach().cpu().numpy().T


SMALL = {
    "cfg1": synth.CONFIGS["cfg1"],
    "cfg2s": synth.CONFIGS["cfg2"].scaled((150, 140, 130), (20, 20, 20), (20, 20, 20)),
    "cfg4s": synth.CONFIGS["cfg4"].scaled((300, 280, 64), (100, 100, 50), (30, 30, 12)),
    "cfg5s": synth.CONFIGS["cfg5"].scaled((160, 150, 140), (40, 40, 40), (40, 40, 40)),
}


@pytest.mark.parametrize("name", list(SMALL))
def test_hosvd_parity(P, h, name):
    cfg = SMALL[name]
    x = synth.make_tensor(cfg)
    oms = _omegas_for(cfg)
    ref = oracle.hosvd(x, cfg.ranks, oms, q=cfg.q)
    res = P.rtucker_hosvd(h, dev(x), cfg.ranks, cfg.p, cfg.q, _to_dev_omegas(oms, "gauss"))
    h.sync()
    _check_result(res, ref, cfg)


@pytest.mark.parametrize("name", list(SMALL))
def test_hosvd_parity_strict_fp64_accumulation(P, name):
    """The strict reference-precision mode (RT_OPT_TTM_IMPL = 3: every X pass accumulates in fp64)
    on the same cases: same metrics, and the sketches to 1e-12 of the oracle's."""
    cfg = SMALL[name]
    x = synth.make_tensor(cfg)
    oms = _omegas_for(cfg)
    ref = oracle.hosvd(x, cfg.ranks, oms, q=cfg.q)
    hh = P.Handle()
    hh.set_option(0, 3)
    try:
        res = P.rtucker_hosvd(hh, dev(x), cfg.ranks, cfg.p, cfg.q, _to_dev_omegas(oms, "gauss"))
        y0 = P.rtucker_sketch(hh, dev(x), 0, om_dev(oms[0]))
        hh.sync()
        _check_result(res, ref, cfg)
        assert M.rel_fro(mat(y0), ref["Y0"][0]) <= 1e-12
    finally:
        hh.close()


def test_sthosvd_kron_parity(P, h):
    cfg = synth.CONFIGS["cfg3"].scaled((40, 36, 32, 30), (6, 6, 6, 6), (6, 6, 6, 6))
    x = synth.make_tensor(cfg)
    oms = _omegas_for(cfg, "kron", sthosvd=True)
    ref = oracle.sthosvd(x, cfg.ranks, oms, q=cfg.q, kind="kron")
    res = P.rtucker_sthosvd(h, dev(x), cfg.ranks, cfg.p, cfg.q, _to_dev_omegas(oms, "kron"), kind="kron")
    h.sync()
    _check_result(res, ref, cfg)


def test_sthosvd_gauss_power_order(P, h):
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"].scaled((70, 60, 50), (8, 8, 8), (8, 8, 8)), q=1)
    x = synth.make_tensor(cfg)
    order = [2, 0, 1]
    N = 3
    d = list(cfg.dims)
    oms = [None] * N
    for n in order:
        J = int(np.prod([d[k] for k in range(N) if k != n]))
        K = min(cfg.ranks[n] + cfg.p, d[n], J)
        oms[n] = np.ascontiguousarray(synth.rng_for(9, 9, n).standard_normal((J, K)).astype(np.float32))
        d[n] = cfg.ranks[n]
    ref = oracle.sthosvd(x, cfg.ranks, oms, q=1, mode_order=order)
    res = P.rtucker_sthosvd(h, dev(x), cfg.ranks, cfg.p, 1, _to_dev_omegas(oms, "gauss"), mode_order=order)
    h.sync()
    _check_result(res, ref, cfg)


def test_hosvd_kron_power(P, h):
    cfg = dataclasses.replace(synth.CONFIGS["cfg3"].scaled((34, 32, 30, 28), (5, 5, 5, 5), (5, 5, 5, 5)), q=1)
    x = synth.make_tensor(cfg)
    oms = _omegas_for(cfg, "kron")
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1, kind="kron")
    res = P.rtucker_hosvd(h, dev(x), cfg.ranks, cfg.p, 1, _to_dev_omegas(oms, "kron"), kind="kron")
    h.sync()
    _check_result(res, ref, cfg)


# ------------------------------------------------------------------ edge cases
def test_zero_tensor(P, h):
    """Reading R7: all-zero X -> Q_n = I[:, :R_n], G = 0, E = 0."""
    dims, ranks, p = (20, 15, 10), (3, 2, 4), 2
    x = np.zeros(dims, dtype=np.float32, order="F")
    rng = np.random.default_rng(10)
    oms = [rng.standard_normal((x.size // dims[n], ranks[n] + p)).astype(np.float32) for n in range(3)]
    res = P.rtucker_hosvd(h, dev(x), ranks, p, 1, [om_dev(o) for o in oms])
    h.sync()
    for n in range(3):
        np.testing.assert_array_equal(mat(res["Q"][n]), np.eye(dims[n], ranks[n]))
    assert np.all(P_core(res["G"]) == 0)
    assert np.all(mat(res["err"]) == 0)


def test_full_rank_and_exact_recovery(P, h):
    """P6 / P4 on the GPU: full rank keeps ||G|| = ||X||; exact rank is recovered to fp32 level."""
    dims = (12, 10, 8)
    x = rand_tensor(11, dims, np.float64)
    rng = np.random.default_rng(12)
    oms = [rng.standard_normal((x.size // dims[n], dims[n])) for n in range(3)]
    res = P.rtucker_hosvd(h, dev(x), dims, 0, 0, [om_dev(o) for o in oms])
    h.sync()
    g = P_core(res["G"])
    assert abs(np.linalg.norm(g) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    assert mat(res["err"])[0] <= 1e-12
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"].scaled((64, 60, 56), (5, 4, 3), (5, 4, 3)), noise="none")
    x = synth.make_tensor(cfg)
    res = P.rtucker_hosvd(h, dev(x), cfg.ranks, 3, 0, [om_dev(synth.gaussian_omega(cfg, n, K=r + 3))
                                                        for n, r in enumerate(cfg.ranks)])
    h.sync()
    assert mat(res["err"])[0] <= 1e-5


def test_rank_one_and_unit_mode(P, h):
    dims = (33, 1, 17)
    x = rand_tensor(13, dims)
    ranks = (1, 1, 1)
    rng = np.random.default_rng(14)
    Ks = [min(1 + 2, dims[n], x.size // dims[n]) for n in range(3)]
    oms = [rng.standard_normal((x.size // dims[n], Ks[n])).astype(np.float32) for n in range(3)]
    ref = oracle.hosvd(x, ranks, oms)
    res = P.rtucker_hosvd(h, dev(x), ranks, 2, 0, [om_dev(o) for o in oms])
    h.sync()
    assert abs(mat(res["err"])[0] - ref["E"]) / ref["E"] <= 1e-5


def test_invalid_arguments(P, h):
    from paper_2001_07124_b200 import RtError
    x = dev(rand_tensor(15, (10, 9, 8)))
    om = om_dev(np.zeros((72, 5), dtype=np.float32))
    with pytest.raises(RtError) as e:
        P.rtucker_sketch(h, x, 3, om)
    assert e.value.status == -1
    with pytest.raises(RtError) as e:            # K > I_n with power iterations (QR needs K <= I_n)
        P.rtucker_sketch(h, x, 0, om_dev(np.zeros((72, 11), dtype=np.float32)), q=1)
    assert e.value.status == -2
    with pytest.raises(RtError) as e:            # R_n > K_n
        P.rtucker_hosvd(h, x, (6, 2, 2), 0, 0, [om, om_dev(np.zeros((80, 2), np.float32)),
                                                om_dev(np.zeros((90, 2), np.float32))])
    assert e.value.status in (-1, -2)
    h.sync()


def test_nonfinite_input_reported(P, h):
    from paper_2001_07124_b200 import RtError
    x = rand_tensor(16, (10, 9, 8))
    x[3, 4, 5] = np.nan
    P.rtucker_sketch(h, dev(x), 0, om_dev(np.ones((72, 4), dtype=np.float32)))
    with pytest.raises(RtError) as e:
        h.sync()
    assert e.value.status == -6


# ----------------------------------------------------------- slab emulation
def test_slab_partial_sums_equal_unsharded(P, h):
    """P18 on the GPU: per-slab sketches/cores (no communicator => partial sums) add up."""
    dims = (23, 19, 31)
    x = rand_tensor(17, dims)
    rng = np.random.default_rng(18)
    slabs = [(0, 10), (10, 11), (11, 31)]
    for n in range(3):
        J = x.size // dims[n]
        om = rng.standard_normal((J, 6)).astype(np.float32)
        full = mat(P.rtucker_sketch(h, dev(x), n, om_dev(om)))
        parts = []
        for lo, hi in slabs:
            xs = np.asfortranarray(x[:, :, lo:hi])
            if n < 2:
                a = dims[0] * dims[1] // dims[n]
                oml = om[a * lo:a * hi]
                parts.append(mat(P.rtucker_sketch(h, dev(xs), n, om_dev(oml), last_offset=lo, last_global=31)))
            else:
                parts.append(mat(P.rtucker_sketch(h, dev(xs), n, om_dev(om), last_offset=lo, last_global=31)))
        got = sum(parts) if n < 2 else np.concatenate(parts, axis=0)
        assert M.rel_fro(got, full) <= 1e-6
    h.sync()


def _run_loopback(P, x, cfg, oms, nranks, bounds, options=()):
    grp = P.LoopbackGroup(nranks)
    out = [None] * nranks
    errs = []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                hh = P.Handle(stream=s, loopback_group=grp, rank=r)
                for o, v in options:
                    hh.set_option(o, v)
                lo, hi = bounds[r]
                xs = dev(np.asfortranarray(x[:, :, lo:hi]))
                loc = []
                for n in range(3):
                    if n < 2:
                        a = cfg.dims[0] * cfg.dims[1] // cfg.dims[n]
                        loc.append(om_dev(oms[n][a * lo:a * hi]))
                    else:
                        loc.append(om_dev(oms[n]))
                res = P.rtucker_hosvd(hh, xs, cfg.ranks, cfg.p, cfg.q, loc, last_offset=lo,
                                      last_global=cfg.dims[2])
                hh.sync()
                out[r] = dict(Q=[mat(q) for q in res["Q"]], G=P_core(res["G"]), err=mat(res["err"]))
                hh.close()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    return out


@pytest.mark.parametrize("nranks", [2, 3])
def test_loopback_multirank_hosvd(P, h, nranks):
    """The full multi-rank control flow (C1-C5) on one GPU: slabs of the last mode on
    `nranks` emulated ranks reproduce the single-rank result; replicated outputs agree."""
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled((48, 40, 36), (6, 6, 6), (6, 6, 6)), q=1)
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    cuts = np.linspace(0, cfg.dims[2], nranks + 1).astype(int)
    bounds = [(int(cuts[r]), int(cuts[r + 1])) for r in range(nranks)]
    out = _run_loopback(P, x, cfg, oms, nranks, bounds)
    for r in range(1, nranks):
        np.testing.assert_array_equal(out[r]["G"], out[0]["G"])
        for n in range(2):
            np.testing.assert_array_equal(out[r]["Q"][n], out[0]["Q"][n])
    q_last = np.concatenate([out[r]["Q"][2] for r in range(nranks)], axis=0)
    qg = out[0]["Q"][:2] + [q_last]
    for n in range(3):
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert M.recon(out[0]["G"], qg, ref["G"], ref["Q"]) <= 1e-5
    assert abs(out[0]["err"][0] - ref["E"]) / ref["E"] <= 1e-5


@pytest.mark.parametrize("nranks,opts", [(2, ()), (3, ()), (2, ((100, 270),)), (3, ((3, 1),)), (2, ((100, 320),)),
                                         (3, ((100, 320), (3, 1)))])
def test_loopback_overlapped_hosvd(P, nranks, opts):
    """The overlapped distributed schedule (K_n % 4 == 0 so every power step takes reading R31): the
    replicated modes' QRs on the side stream, the slab mode's Z allreduce (C3) on the side
    communicator and a third stream while the other modes proceed, then its product from the summed
    Z.  2 and 3 emulated ranks (loopback), with the overlap off (option 270) and with tf32-rounded
    Omega (option 3): the gathered result equals the oracle; replicated outputs agree bit for bit.
    These slabs are thin (I_3(local) < 8 K): by default the slab mode sketches and multiplies with the
    3xTF32 kernels on the fp32 Omega / Z; option 320 keeps the fp16 forms a thick slab takes (Omega
    converted once, the summed Z converted on the C3 stream)."""
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled((48, 40, 36), (6, 6, 6), (6, 6, 6)), q=1, p=10)
    assert all(cfg.K(n) % 4 == 0 for n in range(3))
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    if any(o == 3 for o, _ in opts):
        oms = [synth.round_tf32(o) for o in oms]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    cuts = np.linspace(0, cfg.dims[2], nranks + 1).astype(int)
    out = _run_loopback(P, x, cfg, oms, nranks, [(int(cuts[r]), int(cuts[r + 1])) for r in range(nranks)], opts)
    for r in range(1, nranks):
        np.testing.assert_array_equal(out[r]["G"], out[0]["G"])
        for n in range(2):
            np.testing.assert_array_equal(out[r]["Q"][n], out[0]["Q"][n])
    qg = out[0]["Q"][:2] + [np.concatenate([out[r]["Q"][2] for r in range(nranks)], axis=0)]
    for n in range(3):
        assert M.orth(qg[n]) <= 1e-12
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5, (n, M.subspace(qg[n], ref["Q"][n]))
    assert M.recon(out[0]["G"], qg, ref["G"], ref["Q"]) <= 1e-5
    assert abs(out[0]["err"][0] - ref["E"]) / ref["E"] <= 1e-5


@pytest.mark.parametrize("nranks,opts", [(2, ()), (3, ()), (2, ((100, 350),)), (2, ((100, 212),))])
def test_loopback_slab_residual(P, nranks, opts):
    """The slab form of the residual pass: with a wide sketch (K = 72 > 64) and
    a thin slab, a slab-parallel HOSVD rebuilds X^ slice by slice of the slab mode from
    P' = G x_3 Q_3[local] x_1 Q_1 (J' x K_2 x I_3(local)) with mode 2 contracted in the kernel,
    instead of from the whole J x K_3 tensor P on every rank.  E against the oracle at 1e-5, with
    the old form (option 350) and with the fp16 gate closed (option 212: the SIMT twin in its
    sliced form); replicated outputs agree bit for bit."""
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled((96, 88, 80), (64, 64, 64), (64, 64, 64)), q=1, p=8)
    assert all(cfg.K(n) == 72 for n in range(3))
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    cuts = np.linspace(0, cfg.dims[2], nranks + 1).astype(int)
    out = _run_loopback(P, x, cfg, oms, nranks, [(int(cuts[r]), int(cuts[r + 1])) for r in range(nranks)], opts)
    for r in range(1, nranks):
        np.testing.assert_array_equal(out[r]["G"], out[0]["G"])
        np.testing.assert_array_equal(out[r]["err"], out[0]["err"])
    qg = out[0]["Q"][:2] + [np.concatenate([out[r]["Q"][2] for r in range(nranks)], axis=0)]
    for n in range(3):
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5, (n, M.subspace(qg[n], ref["Q"][n]))
    assert M.recon(out[0]["G"], qg, ref["G"], ref["Q"]) <= 1e-5
    assert abs(out[0]["err"][0] - ref["E"]) / ref["E"] <= 1e-5, (out[0]["err"][0], ref["E"])
