"""Pins of the fp64 oracle against what the paper and the mathematics fix
(SURVEY.md §8(c.4) P1-P20).  CPU only; none of these compare the oracle with
itself -- each checks a worked example, a closed form, an invariant, a
textbook/library routine, or brute force on tiny inputs.
"""
import itertools
import math
import os

import numpy as np
import pytest

import oracle
from gen import synth
from tests import _metrics as M


def _rng(seed):
    return np.random.default_rng(seed)


def _low_rank(rng, dims, ranks, noise=0.0, orth=True):
    g = rng.standard_normal(ranks)
    fs = []
    for d, r in zip(dims, ranks):
        a = rng.standard_normal((d, r))
        fs.append(np.linalg.qr(a)[0] if orth else a)
    x = g
    for n, u in enumerate(fs):
        x = np.moveaxis(np.tensordot(u, x, axes=([1], [n])), 0, n)
    if noise:
        nz = rng.standard_normal(dims)
        x = x + noise * np.linalg.norm(x) / np.linalg.norm(nz) * nz
    return x, g, fs


def _omegas(rng, dims, K):
    N = len(dims)
    return [rng.standard_normal((int(np.prod([d for k, d in enumerate(dims) if k != n])), K[n]))
            for n in range(N)]


# ------------------------------------------------------------------ P1, P17
def test_P1_unfold_worked_example(golden_dir):
    """P1: SPEC.md S:62 worked example of the §II j-index."""
    rows = [list(map(float, l.split())) for l in open(os.path.join(golden_dir, "unfold_2x2x2.txt"))
            if l.strip() and not l.startswith("#")]
    t = np.zeros((2, 2, 2))
    for i, j, k in itertools.product(range(2), repeat=3):
        t[i, j, k] = 100 * (i + 1) + 10 * (j + 1) + (k + 1)
    np.testing.assert_array_equal(oracle.unfold(t, 0), np.array(rows))


def test_P1b_unfold_matches_j_index_formula_by_loops():
    """Brute force of the §II formula j = sum_{k!=n} i_k J_k, J_k = prod_{m<k,m!=n} I_m."""
    rng = _rng(1)
    for dims in [(3, 4, 2), (2, 3, 2, 3), (5, 1, 3)]:
        x = rng.standard_normal(dims)
        for n in range(len(dims)):
            u = oracle.unfold(x, n)
            assert u.shape == (dims[n], x.size // dims[n])
            for idx in itertools.product(*[range(d) for d in dims]):
                j, Jk = 0, 1
                for k in range(len(dims)):
                    if k == n:
                        continue
                    j += idx[k] * Jk
                    Jk *= dims[k]
                assert u[idx[n], j] == x[idx]
            np.testing.assert_array_equal(oracle.fold(u, n, dims), x)


def test_P17_ttm_and_sketch_brute_force():
    """P17: n-mode product and Gaussian sketch (Eq. proj) by loops."""
    rng = _rng(2)
    dims = (3, 4, 2)
    x = rng.standard_normal(dims)
    for n in range(3):
        b = rng.standard_normal((5, dims[n]))
        ref = np.zeros(tuple(5 if k == n else d for k, d in enumerate(dims)))
        for idx in itertools.product(*[range(d) for d in ref.shape]):
            s = 0.0
            for i in range(dims[n]):
                src = list(idx)
                src[n] = i
                s += x[tuple(src)] * b[idx[n], i]
            ref[idx] = s
        np.testing.assert_allclose(oracle.ttm(x, b, n), ref, rtol=1e-14, atol=1e-14)
        # sketch Y = X_(n) Omega with Omega rows in j-index order, by loops
        J = x.size // dims[n]
        om = rng.standard_normal((J, 3))
        y0, _ = oracle.sketch_gauss(x, n, om, 0)
        others = [k for k in range(3) if k != n]
        yref = np.zeros((dims[n], 3))
        for i in range(dims[n]):
            for a in range(dims[others[0]]):
                for c in range(dims[others[1]]):
                    j = a + dims[others[0]] * c
                    src = [0, 0, 0]
                    src[n], src[others[0]], src[others[1]] = i, a, c
                    yref[i] += x[tuple(src)] * om[j]
        np.testing.assert_allclose(y0, yref, rtol=1e-13, atol=1e-13)


# ------------------------------------------------------------------ P2, P3
def test_P2_eq1_same_mode_products():
    """P2: Eq.(1) X x_n B x_n A = X x_n (AB)."""
    rng = _rng(3)
    x = rng.standard_normal((4, 5, 6))
    for n in range(3):
        b = rng.standard_normal((7, x.shape[n]))
        a = rng.standard_normal((3, 7))
        lhs = oracle.ttm(oracle.ttm(x, b, n), a, n)
        rhs = oracle.ttm(x, a @ b, n)
        assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)


def test_P3_eq2_kron_sketch_equals_kronecker_product():
    """P3: Kronecker sketch W_(n) = X_(n)(Omega_N kron ... kron Omega_1, without n),
    Eq.(2) P:118-130 with numpy.kron as the independent routine."""
    rng = _rng(4)
    for dims in [(4, 5, 3), (3, 4, 2, 5)]:
        x = rng.standard_normal(dims)
        N = len(dims)
        for n in range(N):
            oms = [None if k == n else rng.standard_normal((dims[k], 2 + k % 2)) for k in range(N)]
            y0, _ = oracle.sketch_kron(x, n, oms, 0)
            kr = np.ones((1, 1))
            for k in reversed(range(N)):
                if k != n:
                    kr = np.kron(kr, oms[k])
            ref = oracle.unfold(x, n) @ kr
            assert np.linalg.norm(y0 - ref) <= 1e-12 * np.linalg.norm(ref)


def test_P3b_eq2_tucker_unfold():
    """Eq.(2): X = S x_1 Q1 ... => X_(n) = Q_n S_(n) (Q_N kron .. kron Q_1 without n)^T."""
    rng = _rng(5)
    s = rng.standard_normal((2, 3, 2))
    qs = [rng.standard_normal((d, r)) for d, r in zip((4, 5, 3), s.shape)]
    x = oracle.reconstruct(s, qs)
    for n in range(3):
        kr = np.ones((1, 1))
        for k in reversed(range(3)):
            if k != n:
                kr = np.kron(kr, qs[k])
        ref = qs[n] @ oracle.unfold(s, n) @ kr.T
        np.testing.assert_allclose(oracle.unfold(x, n), ref, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------- QR / EVD
def test_qr_plus_matches_gram_schmidt_by_loops():
    """qr+ (R_ii >= 0) equals classical Gram-Schmidt with reorthogonalization."""
    rng = _rng(6)
    y = rng.standard_normal((30, 6))
    q, r = oracle.qr_plus(y)
    qg = np.zeros_like(y)
    for c in range(6):
        v = y[:, c].copy()
        for _ in range(2):
            for l in range(c):
                v -= (qg[:, l] @ v) * qg[:, l]
        qg[:, c] = v / np.linalg.norm(v)
    np.testing.assert_allclose(q, qg, atol=1e-13)
    assert np.all(np.diag(r) >= 0)
    np.testing.assert_allclose(q @ r, y, atol=1e-13)


def test_eig_desc_recovers_constructed_spectrum():
    rng = _rng(7)
    v, _ = np.linalg.qr(rng.standard_normal((8, 8)))
    lam = np.array([9.0, 7.5, 5.0, 3.0, 2.0, 1.0, 0.5, 0.1])
    m = (v * lam) @ v.T
    w, u = oracle.eig_desc(m)
    np.testing.assert_allclose(w, lam, rtol=1e-13)
    for c in range(8):
        assert abs(abs(u[:, c] @ v[:, c]) - 1) < 1e-12


def test_canon_sign_rule():
    """Reading R5: largest-|.| entry positive, lowest row on ties."""
    qn = np.array([[0.1, -0.5], [-0.9, 0.5], [0.2, 0.1]])
    u = np.eye(2)
    q2, u2 = oracle.canon_sign(qn, u)
    np.testing.assert_array_equal(q2[:, 0], -qn[:, 0])     # max |.| at row 1 is negative
    np.testing.assert_array_equal(q2[:, 1], -qn[:, 1])     # tie rows 0/1 -> row 0 (-0.5) flips
    np.testing.assert_array_equal(u2, np.diag([-1.0, -1.0]))


# ------------------------------------------------------------------ P4-P10
@pytest.mark.parametrize("kind", ["gauss", "kron"])
def test_P4_P5_exact_rank_recovery(kind):
    """P4/P5: exact multilinear rank, noise-free, K_n >= R_n => E < 1e-10 and
    ||Q^TQ - I|| < 1e-12 (BASELINE north_star; Table I row 1 magnitudes P:908)."""
    rng = _rng(8)
    dims, ranks = (30, 25, 20), (4, 3, 5)
    x, _, _ = _low_rank(rng, dims, ranks)
    if kind == "gauss":
        oms = _omegas(rng, dims, [r + 3 for r in ranks])
    else:
        oms = [[None if k == n else rng.standard_normal((dims[k], 3)) for k in range(3)] for n in range(3)]
    res = oracle.hosvd(x, ranks, oms, q=0, kind=kind)
    assert res["E"] < 1e-10
    for qn in res["Q"]:
        assert np.linalg.norm(qn.T @ qn - np.eye(qn.shape[1])) < 1e-12
    # R-STHOSVD on the same input: sketch matrices sized for the shrinking tensor
    d = list(dims)
    oms2 = []
    for n in range(3):
        if kind == "gauss":
            J = int(np.prod([d[k] for k in range(3) if k != n]))
            oms2.append(rng.standard_normal((J, ranks[n] + 3)))
        else:
            oms2.append([None if k == n else rng.standard_normal((d[k], 3)) for k in range(3)])
        d[n] = ranks[n]
    res2 = oracle.sthosvd(x, ranks, oms2, q=0, kind=kind)
    assert res2["E"] < 1e-10


def test_P6_full_rank_norm_preserved():
    """P6: R_n = I_n, p = 0 => ||G||_F = ||X||_F and E ~ 0 (TK1 P:397-400)."""
    rng = _rng(9)
    dims = (6, 5, 4)
    x = rng.standard_normal(dims)
    oms = _omegas(rng, dims, list(dims))
    res = oracle.hosvd(x, dims, oms)
    assert abs(oracle.fro(res["G"]) - oracle.fro(x)) <= 1e-13 * oracle.fro(x)
    assert res["E"] < 1e-13


def _align(a, b):
    s = np.sign(np.sum(a * b, axis=0))
    s[s == 0] = 1
    return a * s


def test_P7_full_sketch_equals_deterministic_thosvd():
    """P7: K_n = I_n => randomized HOSVD == deterministic THOSVD via full SVD of each
    unfolding, factors and core, when signs follow R5 on the lifted factor."""
    rng = _rng(10)
    dims, ranks = (7, 6, 5), (3, 2, 4)
    x = rng.standard_normal(dims)
    oms = _omegas(rng, dims, list(dims))
    res = oracle.hosvd(x, ranks, oms)
    ref = oracle.thosvd(x, ranks)
    for a, b in zip(res["Q"], ref["Q"]):
        np.testing.assert_allclose(a, b, atol=1e-12)
    np.testing.assert_allclose(res["G"], ref["G"], atol=1e-12)
    assert abs(res["E"] - ref["E"]) < 1e-12


def test_P7_full_sketch_equals_deterministic_sthosvd():
    """P7 for Alg.8 vs Alg.4: K_n = current I_n => R-STHOSVD == STHOSVD."""
    rng = _rng(11)
    dims, ranks = (7, 6, 5), (3, 2, 4)
    x = rng.standard_normal(dims)
    d = list(dims)
    oms = []
    for n in range(3):
        J = int(np.prod([d[k] for k in range(3) if k != n]))
        oms.append(rng.standard_normal((J, d[n])))
        d[n] = ranks[n]
    res = oracle.sthosvd(x, ranks, oms)
    ref = oracle.sthosvd_det(x, ranks)
    for a, b in zip(res["Q"], ref["Q"]):
        np.testing.assert_allclose(a, b, atol=1e-12)
    np.testing.assert_allclose(res["G"], ref["G"], atol=1e-12)


def test_P8_P9_pythagoras_and_subpro():
    """P8: E^2 = 1 - ||G||^2/||X||^2; P9: SubPro bound."""
    rng = _rng(12)
    dims, ranks = (20, 18, 16), (4, 4, 4)
    x, _, _ = _low_rank(rng, dims, ranks, noise=0.3)
    oms = _omegas(rng, dims, [6, 6, 6])
    res = oracle.hosvd(x, ranks, oms, q=1)
    e2 = res["E"] ** 2
    assert abs(e2 - (1 - oracle.fro(res["G"]) ** 2 / oracle.fro(x) ** 2)) < 1e-13
    # the oracle's E_gram diagnostic is this identity: equal to the direct residual E
    # (a dropped square or sqrt in rel_error_gram fails here: E ~ 0.3 is far from E^2 and sqrt(E))
    assert abs(res["E_gram"] - res["E"]) < 1e-12
    assert abs(oracle.rel_error_gram(x, res["G"]) - res["E"]) < 1e-12
    # closed forms: ||X|| = 5, ||G|| = 3 -> sqrt(1 - 9/25) = 0.8; ||G|| >= ||X|| -> 0; X = 0 -> 0
    x5 = np.zeros((2, 2, 2)); x5[0, 0, 0], x5[1, 1, 1] = 3.0, 4.0
    g3 = np.zeros((1, 1, 1)); g3[0, 0, 0] = 3.0
    assert abs(oracle.rel_error_gram(x5, g3) - 0.8) < 1e-15
    assert oracle.rel_error_gram(x5, 2 * g3) == 0.0
    assert oracle.rel_error_gram(np.zeros((2, 2, 2)), g3) == 0.0
    bound = 0.0
    for n, qn in enumerate(res["Q"]):
        xn = oracle.unfold(x, n)
        bound += np.linalg.norm(xn - qn @ (qn.T @ xn)) ** 2
    assert (res["E"] * oracle.fro(x)) ** 2 <= bound * (1 + 1e-12)


def test_P10_all_orthogonal_core_when_lossless():
    """P10: exact rank and K_n >= R_n => all-orthogonal, pseudo-diagonal core."""
    rng = _rng(13)
    dims, ranks = (15, 14, 13), (4, 3, 5)
    x, _, _ = _low_rank(rng, dims, ranks)
    res = oracle.hosvd(x, ranks, _omegas(rng, dims, [r + 2 for r in ranks]))
    g = res["G"]
    for n in range(3):
        gn = oracle.unfold(g, n)
        m = gn @ gn.T
        off = m - np.diag(np.diag(m))
        assert np.linalg.norm(off) <= 1e-12 * np.linalg.norm(m)
        d = np.diag(m)
        assert np.all(np.diff(d) <= 1e-12 * d[0])


def test_R7_zero_input():
    dims, ranks = (5, 4, 3), (2, 2, 2)
    res = oracle.hosvd(np.zeros(dims), ranks, [None] * 3)
    assert res["E"] == 0.0 and np.all(res["G"] == 0)
    for qn, r in zip(res["Q"], ranks):
        np.testing.assert_array_equal(qn, np.eye(qn.shape[0], r))


# ------------------------------------------------------------ statistical pins
def _svd_matrix(rng, m, n, sig):
    u, _ = np.linalg.qr(rng.standard_normal((m, len(sig))))
    v, _ = np.linalg.qr(rng.standard_normal((n, len(sig))))
    return (u * sig) @ v.T


def test_P11_rsvd_expectation_bound():
    """P11: E||X - QQ^TX||_2 <= (1 + sqrt(R/(P-1)) + e sqrt(R+P)/P sqrt(min(I,J)-R))^{1/(2q+1)} sigma_{R+1}
    (reading R13), averaged over 100 Gaussian test matrices."""
    rng = _rng(14)
    m, n, R, P = 60, 80, 6, 4
    sig = 1.0 / np.arange(1, 61) ** 0.5
    x = _svd_matrix(rng, m, n, sig)
    for q in (0, 1):
        errs = []
        for s in range(100):
            om = np.random.default_rng(1000 + s).standard_normal((n, R + P))
            _, y = oracle.sketch_gauss(x, 0, om, q)
            qm, _ = oracle.qr_plus(y)
            errs.append(np.linalg.norm(x - qm @ (qm.T @ x), 2))
        bound = (1 + math.sqrt(R / (P - 1)) + math.e * math.sqrt(R + P) / P * math.sqrt(min(m, n) - R)) \
            ** (1.0 / (2 * q + 1)) * sig[R]
        assert np.mean(errs) <= bound
        assert min(errs) >= sig[R + P] * (1 - 1e-12)    # Eckart-Young: rank R+P projector


def test_P20_power_iteration_span_equals_closed_form():
    """Alg.1 line 2: span Y = span (XX^T)^q X Omega; the sequential QR form (P:212,
    reading R2) must give the same subspace on a well-conditioned case."""
    rng = _rng(15)
    x = _svd_matrix(rng, 40, 50, np.linspace(3.0, 1.0, 40))
    om = rng.standard_normal((50, 5))
    for q in (1, 2):
        _, y = oracle.sketch_gauss(x, 0, om, q)
        ref = np.linalg.matrix_power(x @ x.T, q) @ x @ om
        qa, _ = np.linalg.qr(y)
        qb, _ = np.linalg.qr(ref)
        assert np.linalg.norm(qa @ qa.T - qb @ qb.T) < 1e-10


def test_P15_more_power_iterations_lower_error():
    """P15: q up => mean E down on a slow-decay input (Remark 1)."""
    rng = _rng(16)
    dims, ranks = (24, 22, 20), (4, 4, 4)
    x, _, _ = _low_rank(rng, dims, (12, 12, 12))
    x = x + 0.05 * np.linalg.norm(x) / math.sqrt(x.size) * rng.standard_normal(dims)
    means = []
    for q in (0, 1, 2):
        es = [oracle.hosvd(x, ranks, _omegas(np.random.default_rng(50 + s), dims, [5, 5, 5]), q=q)["E"]
              for s in range(8)]
        means.append(np.mean(es))
    assert means[0] > means[1] > means[2] * (1 - 1e-9)


def test_P12_quasi_optimality():
    """P12: ||X - THOSVD|| <= sqrt(N) ||X - X_best|| with HOOI as X_best proxy."""
    rng = _rng(17)
    for s in range(5):
        x = rng.standard_normal((8, 7, 6))
        e_t = oracle.thosvd(x, (3, 3, 3))["E"]
        e_h = oracle.hooi(x, (3, 3, 3), iters=30)["E"]
        assert e_t <= math.sqrt(3) * e_h + 1e-12
        assert e_h <= e_t + 1e-12


# ------------------------------------------------------------ P13, P14, P16, P19
def test_P13_noise_scaling():
    """P13: realized ||gamma N||/||X_s|| = rho, SNR = -20 log10 rho (reading R11)."""
    cfg = synth.CONFIGS["cfg2"].scaled((20, 18, 16), (3, 3, 3), (3, 3, 3))
    import dataclasses
    cfg = dataclasses.replace(cfg, dtype="f64")
    x, xs, core, factors, gamma = synth.make_tensor(cfg, return_parts=True)
    rho = oracle.fro(x - xs) / oracle.fro(xs)
    assert abs(rho - cfg.noise_level) <= 1e-12
    snr = 10 * math.log10(oracle.fro(xs) ** 2 / oracle.fro(x - xs) ** 2)
    assert abs(snr - 40.0) < 1e-9
    assert abs(oracle.fro(xs) - oracle.fro(core)) <= 1e-12 * oracle.fro(core)   # orthonormal factors


def test_P14_table3_compression(golden_dir):
    """P14: Table III "1/Compression ratio" column from P:839-843."""
    dims = (2200, 1080, 1980)
    for line in open(os.path.join(golden_dir, "table3_compression.txt")):
        if not line.strip() or line.startswith("#"):
            continue
        r, printed, _ = line.split()
        val = synth.compression_inverse(dims, (int(r),) * 3)
        # tolerance: half a unit in the last printed digit
        mant = printed.split("e")[0]
        decimals = len(mant.split(".")[1]) if "." in mant else 0
        exp = int(printed.split("e")[1]) if "e" in printed else 0
        assert abs(val - float(printed)) <= 0.5 * 10.0 ** (exp - decimals) + 1e-15


def test_P16_sthosvd_shortcut_equals_mode_products():
    """P16: S = B x_n U^T equals S x_n Q_n^T (Eq.(1)): the final core of
    R-STHOSVD equals X x_1 Q_1^T ... x_N Q_N^T."""
    rng = _rng(18)
    dims, ranks = (12, 10, 9), (3, 4, 2)
    x, _, _ = _low_rank(rng, dims, (5, 5, 5), noise=0.1)
    d = list(dims)
    oms = []
    for n in range(3):
        J = int(np.prod([d[k] for k in range(3) if k != n]))
        oms.append(rng.standard_normal((J, ranks[n] + 2)))
        d[n] = ranks[n]
    res = oracle.sthosvd(x, ranks, oms, q=1)
    g2 = oracle.core(x, res["Q"])
    assert np.linalg.norm(res["G"] - g2) <= 1e-12 * np.linalg.norm(g2)


def test_P19_noise_floor_error():
    """P19: exact rank + rho-relative white noise => E ~ rho/sqrt(1+rho^2) (derived)."""
    cfg = synth.CONFIGS["cfg2"].scaled((60, 60, 60), (5, 5, 5), (5, 5, 5))
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    res = oracle.hosvd(x, cfg.ranks, oms, q=cfg.q)
    rho = cfg.noise_level
    assert abs(res["E"] / (rho / math.sqrt(1 + rho * rho)) - 1) < 0.02


def test_generators_deterministic_and_slab_consistent():
    cfg = synth.CONFIGS["cfg2"].scaled((9, 8, 7), (2, 2, 2), (2, 2, 2))
    a = synth.make_tensor(cfg)
    b = synth.make_tensor(cfg)
    assert np.array_equal(a, b) and a.flags.f_contiguous
    om = synth.gaussian_omega(cfg, 1)
    part = synth.gaussian_omega(cfg, 1, rows=20, row0=13)
    assert np.array_equal(om[13:33], part)


# ----------------------------------------------------------------- R-PET (Alg.9)
def _lowrank(seed, dims, r):
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((r,) * len(dims))
    us = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d in dims]
    return oracle.reconstruct(g, us), us


def test_P21_pet_exact_rank_recovery():
    """Alg.9 with K = 2R, S = 2K + 1 recovers an exact multilinear-rank-R tensor."""
    dims, r = (30, 28, 26), 4
    x, us = _lowrank(21, dims, r)
    rng = np.random.default_rng(22)
    ks = [2 * r] * 3
    ss = [2 * k + 1 for k in ks]
    oms = [rng.standard_normal((x.size // d, k)) for d, k in zip(dims, ks)]
    omt = [rng.standard_normal((s_, d)) for s_, d in zip(ss, dims)]
    out = oracle.pet(x, (r,) * 3, oms, omt)
    assert out["E"] < 1e-8
    for n in range(3):
        assert np.linalg.norm(out["Q"][n].T @ out["Q"][n] - np.eye(r)) < 1e-12
        p = out["Q"][n] @ out["Q"][n].T
        assert np.linalg.norm(p @ us[n] - us[n]) < 1e-8            # captured the true factor


def test_P22_pet_core_recovery_inverts_the_core_sketch():
    """Line 4: if X = C x_n Q_n (X inside span(Q)), S = H x_n (Omega~_n Q_n)^+ returns C exactly
    (the pseudo-inverse of a full-column-rank Omega~_n Q_n is a left inverse)."""
    dims, k = (12, 11, 10), 3
    rng = np.random.default_rng(23)
    c = rng.standard_normal((k, k, k))
    qs = [np.linalg.qr(rng.standard_normal((d, k)))[0] for d in dims]
    x = oracle.reconstruct(c, qs)
    omt = [rng.standard_normal((2 * k + 1, d)) for d in dims]
    h = oracle.multi_ttm(x, omt)
    s = oracle.multi_ttm(h, [np.linalg.pinv(o @ q) for o, q in zip(omt, qs)])
    assert np.linalg.norm(s - c) <= 1e-12 * np.linalg.norm(c)


def test_P23_pet_identity_core_sketch_reduces_to_rp_hosvd():
    """With Omega~_n = I_{I_n} (S_n = I_n) line 4 is S = X x_n Q_n^+ = X x_n Q_n^T (orthonormal
    Q), the RP-HOSVD core of Alg.6: R-PET then equals hosvd() on the same Omega_n."""
    cfg = synth.CONFIGS["cfg2"].scaled((20, 18, 16), (3, 3, 3), (3, 3, 3))
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    a = oracle.pet(x, cfg.ranks, oms, [np.eye(d) for d in cfg.dims])
    b = oracle.hosvd(x, cfg.ranks, oms, q=0)
    for n in range(3):
        assert np.linalg.norm(a["Q"][n] - b["Q"][n]) < 1e-10
    assert np.linalg.norm(a["G"] - b["G"]) < 1e-10 * np.linalg.norm(b["G"])
    assert abs(a["E"] - b["E"]) < 1e-12


# ------------------------------------------------------------- Khatri-Rao sketch
def test_P24_khatri_rao_sketch_is_explicit_brute_force():
    """sketch_kr equals X_(n) times the explicit Khatri-Rao matrix built entry by entry:
    row j (first-mode-fastest over k != n, reading R6) of column c is prod_k Omega_k[i_k, c]."""
    dims = (4, 3, 5)
    rng = np.random.default_rng(24)
    x = rng.standard_normal(dims)
    K = 2
    for n in range(3):
        oms = [None if k == n else rng.standard_normal((dims[k], K)) for k in range(3)]
        others = [k for k in range(3) if k != n]
        J = int(np.prod([dims[k] for k in others]))
        kr = np.zeros((J, K))
        for c in range(K):
            for idx in np.ndindex(*[dims[k] for k in reversed(others)]):
                sub = dict(zip(reversed(others), idx))
                j = 0
                stride = 1
                for k in others:                       # first-mode-fastest linearization
                    j += sub[k] * stride
                    stride *= dims[k]
                kr[j, c] = np.prod([oms[k][sub[k], c] for k in others])
        y0, _ = oracle.sketch_kr(x, n, oms)
        brute = np.zeros((dims[n], K))
        for i in range(dims[n]):
            row = np.moveaxis(x, n, 0)[i]
            for c in range(K):
                w = row.copy()
                for pos, k in reversed(list(enumerate(others))):
                    w = np.tensordot(w, oms[k][:, c], axes=([pos], [0]))
                brute[i, c] = w
        assert np.allclose(y0, oracle.unfold(x, n) @ kr, rtol=0, atol=1e-12)
        assert np.allclose(y0, brute, rtol=0, atol=1e-12)


# ----------------------------------------------------------------- RP-HOOI (Alg.7)
def test_P25_rp_hooi_exact_rank_from_random_start():
    """Alg.7 from random orthonormal starting factors recovers an exact multilinear-rank-R
    tensor in one sweep (S_(n) has rank R_n, so orth(S_(n) Omega) spans it): E <= 1e-10."""
    dims, r = (20, 18, 16), 3
    x, us = _lowrank(25, dims, r)
    rng = np.random.default_rng(26)
    q0 = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d in dims]
    oms = [[rng.standard_normal((r * r, r)) for _ in range(3)] for _ in range(2)]
    out = oracle.rp_hooi(x, (r,) * 3, q0, oms)
    assert out["E"] <= 1e-10
    for n in range(3):
        assert np.linalg.norm(out["Q"][n].T @ out["Q"][n] - np.eye(r)) < 1e-12


def test_P26_rp_hooi_matrix_identity_sketch_is_subspace_iteration():
    """N = 2, R_1 = R_2 = R, Omega^(n) = I_R: line 5 is W = S_(n) = X Q^(2) (resp. X^T Q^(1)), so a
    sweep is one step of orthogonal (subspace) iteration, i.e. the HOOI update for matrices."""
    rng = np.random.default_rng(27)
    x = rng.standard_normal((30, 25))
    r = 4
    q1, q2 = (np.linalg.qr(rng.standard_normal((d, r)))[0] for d in x.shape)
    out = oracle.rp_hooi(x, (r, r), [q1, q2], [[np.eye(r), np.eye(r)]])
    e1 = np.linalg.qr(x @ q2)[0]
    e2 = np.linalg.qr(x.T @ e1)[0]
    # (the projector-distance metric has a ~1e-8 floor: sqrt of an fp64 cancellation)
    assert M.subspace(out["Q"][0], e1) < 1e-7 and M.subspace(out["Q"][1], e2) < 1e-7


def test_P27_rp_hooi_above_the_hooi_optimum():
    """No orthonormal factors beat the (converged) HOOI fit: E_rphooi >= E_hooi (1 - 1e-9)."""
    cfg = synth.CONFIGS["cfg2"].scaled((24, 22, 20), (4, 4, 4), (4, 4, 4))
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    a = oracle.hosvd(x, cfg.ranks, oms, q=0)
    b = oracle.rp_hooi(x, cfg.ranks, a["Q"], synth.hooi_omegas(cfg, 3))
    c = oracle.hooi(x, cfg.ranks)
    assert c["E"] * (1 - 1e-9) <= b["E"]


# ------------------------------------------------------------ count sketch
def _explicit_count_matrix(codes, K):
    """S in {0, +-1}^{J x K} written out entry by entry: S[j, h_j] = s_j."""
    S = np.zeros((len(codes), K))
    for j, v in enumerate(codes):
        S[j, abs(int(v)) - 1] = 1.0 if v > 0 else -1.0
    return S


def test_P28_count_sketch_equals_explicit_sign_hash_matrix():
    """The three-step count sketch (hash, group, signed sum) equals X_(n) S for the explicit
    one-nonzero-per-row sign/hash matrix S, every mode, order 3 and 4, ragged sizes."""
    for dims in [(7, 5, 6), (4, 3, 5, 2)]:
        rng = np.random.default_rng(sum(dims))
        x = rng.standard_normal(dims)
        for n in range(len(dims)):
            J = int(np.prod(dims)) // dims[n]
            K = 3
            codes = ((rng.integers(0, K, J) + 1) * (2 * rng.integers(0, 2, J) - 1)).astype(np.int32)
            y0, _ = oracle.sketch(x, n, "count", (codes, K))
            # X_(n)(i, j) with the Kolda j-index, written as loops over the entries
            xn = np.zeros((dims[n], J))
            for idx in np.ndindex(*dims):
                j, stride = 0, 1
                for k in range(len(dims)):
                    if k == n:
                        continue
                    j += idx[k] * stride
                    stride *= dims[k]
                xn[idx[n], j] = x[idx]
            assert np.allclose(y0, xn @ _explicit_count_matrix(codes, K), atol=1e-13, rtol=0)


def test_P29_count_sketch_permutation_is_column_permutation():
    """K = J with distinct labels and all signs +: Y0 is X_(n) with its columns permuted."""
    rng = np.random.default_rng(29)
    x = rng.standard_normal((6, 4, 5))
    J = 20
    perm = rng.permutation(J)
    y0, _ = oracle.sketch(x, 0, "count", ((perm + 1).astype(np.int32), J))
    xn = x.reshape(6, J, order="F")
    assert np.array_equal(y0[:, perm], xn)


def test_P30_count_sketch_norm_unbiased():
    """E[S S^T] = I for Rademacher signs (footnote P:309): the mean of ||Y0||_F^2 over draws is
    ||X||_F^2 (a dropped sign gives cross terms and fails this by far)."""
    rng = np.random.default_rng(30)
    x = rng.standard_normal((8, 6, 5)) + 1.0                  # non-zero mean: cross terms matter
    J, K, draws = 30, 4, 3000
    acc = 0.0
    for _ in range(draws):
        codes = ((rng.integers(0, K, J) + 1) * (2 * rng.integers(0, 2, J) - 1)).astype(np.int32)
        acc += np.sum(oracle.sketch(x, 0, "count", (codes, K))[0] ** 2)
    assert abs(acc / draws / np.sum(x ** 2) - 1.0) < 0.03


def test_P31_count_sketch_hosvd_exact_rank_recovery():
    """RP-HOSVD with count-sketch operators (K_n = R + p) recovers an exact multilinear-rank
    tensor: the sketch X_(n) S spans range(X_(n)) for generic labels/signs; E < 1e-10."""
    dims, r = (24, 22, 20), 3
    x, _ = _lowrank(31, dims, r)
    cfg = synth.CONFIGS["cfg1"].scaled(dims, (r,) * 3, (r,) * 3)
    oms = [synth.count_codes(cfg, n, K=r + 3) for n in range(3)]
    out = oracle.hosvd(x, (r,) * 3, oms, q=0, kind="count")
    assert out["E"] < 1e-10


# --------------------------------------------------------- P18 (slab-wise oracle)
@pytest.mark.parametrize("dims,ranks,K,q,slab", [((14, 12, 11), (3, 4, 2), (6, 7, 5), 0, 4),
                                                 ((14, 12, 11), (3, 4, 2), (6, 7, 5), 1, 5),
                                                 ((9, 8, 7, 10), (2, 3, 2, 3), (4, 5, 4, 5), 2, 3),
                                                 ((13, 15), (3, 4), (5, 6), 1, 4)])
def test_P18_slabwise_oracle_equals_oracle_hosvd(dims, ranks, K, q, slab):
    """P18: oracle.slabbed.hosvd_slabs (the cfg5-size evaluation of the oracle, tests/
    test_gpu_fullsize.py) splits every sum over the last mode into slab partial sums -- a
    reassociation only, so it equals oracle.hosvd to rounding on any input (ragged last slab)."""
    from oracle.slabbed import hosvd_slabs
    rng = _rng(18)
    x, _, _ = _low_rank(rng, dims, ranks, noise=0.2)
    oms = _omegas(rng, dims, K)
    got = hosvd_slabs(np.asfortranarray(x.astype(np.float32)).astype(np.float64), ranks, oms, q=q, slab=slab)
    ref = oracle.hosvd(np.asfortranarray(x.astype(np.float32)).astype(np.float64), ranks, oms, q=q)
    for n in range(len(dims)):
        np.testing.assert_allclose(got["Y0"][n], ref["Y0"][n], rtol=0, atol=1e-12 * np.abs(ref["Y0"][n]).max())
        np.testing.assert_allclose(got["Qt"][n], ref["Qt"][n], rtol=0, atol=1e-11)
        np.testing.assert_allclose(got["Q"][n], ref["Q"][n], rtol=0, atol=1e-11)
    np.testing.assert_allclose(got["G"], ref["G"], rtol=0, atol=1e-11 * np.abs(ref["G"]).max())
    assert abs(got["E"] - ref["E"]) <= 1e-12 * ref["E"]
    assert abs(got["E_gram"] - ref["E_gram"]) <= 1e-10
