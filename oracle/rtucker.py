"""fp64 oracle of the randomized Tucker/HOSVD hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, step-by-step numpy float64 implementation of what the CUDA path
computes, in the paper's order and notation.  It shares no code with the CUDA
path; only ``gen.synth`` (input generation) serves both.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference legs may
use it.

Readings of the paper:
  R1  sketch width K_n = min(R_n+p, I_n, J_n); HOSVD truncates the oversampled
      core by a small HOSVD (Gram-EVD of the core unfoldings); STHOSVD applies
      Alg.1 lines 4-7 through the Gram-EVD of B_(n).
  R2  power iteration: Q = qr+(Y); Z = qr+(X_(n)^T Q); Y = X_(n) Z  (q times).
  R3  Kronecker sketch: Omega_k^{(n)} in R^{d_k x L_k}, Y_n = W_(n), W = S x_{k!=n} Omega_k^T.
  R5  QR with R_ii >= 0; eigenvalues descending; each lifted factor column made
      positive at its largest-|.| entry (lowest row on ties), same flip on the core.
  R7  all-zero input: Q_n = I[:, :R_n], G = 0, E = 0.
  R8  Alg.8 line 1 "S = X_(n)" read as S = X.
  R12 E is measured against the (noisy) input X.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .tensor import fro, fold, multi_ttm, reconstruct, ttm, unfold


# --------------------------------------------------------------------------- QR
def qr_plus(y: np.ndarray):
    """Economic QR Y = Q R with R_ii >= 0 (reading R5).

    Householder QR from LAPACK (numpy.linalg.qr, 'reduced'), then D = sign(diag R)
    with 0 -> +1, Q <- Q D, R <- D R (unique factorization for full column rank).
    """
    q, r = np.linalg.qr(np.asarray(y, dtype=np.float64), mode="reduced")
    d = np.sign(np.diag(r)).copy()
    d[d == 0] = 1.0
    return q * d[None, :], r * d[:, None]


# ----------------------------------------------------------------------- sketch
def sketch_gauss(x: np.ndarray, n: int, omega: np.ndarray, q: int = 0):
    """Gaussian mode-n sketch with q power iterations (Alg.6 line 3 P:556; Eq. proj
    P:166-172; Alg.1 line 2 P:205 with the stable sequential form P:212, reading R2).

    Returns (Y0, Y): the first sketch Y0 = X_(n) Omega and the final Y.
    """
    xn = unfold(np.asarray(x, dtype=np.float64), n)
    y0 = xn @ np.asarray(omega, dtype=np.float64)
    y = y0
    for _ in range(q):
        qy, _ = qr_plus(y)
        z, _ = qr_plus(xn.T @ qy)
        y = xn @ z
    return y0, y


def sketch_kron(x: np.ndarray, n: int, omegas: Sequence[Optional[np.ndarray]], q: int = 0):
    """Kronecker-structured mode-n sketch (reading R3).

    W = X x_k Omega_k^T for all k != n in ascending k; Y0 = W_(n).  By Eq.(2)
     this equals X_(n) (Omega_N kron ... kron Omega_1, without n).
    Power iterations (if q > 0) continue with dense Z exactly as in ``sketch_gauss``.
    """
    w = np.asarray(x, dtype=np.float64)
    for k, om in enumerate(omegas):
        if k == n:
            continue
        w = ttm(w, np.asarray(om, dtype=np.float64).T, k)
    y0 = unfold(w, n)
    y = y0
    if q:
        xn = unfold(np.asarray(x, dtype=np.float64), n)
        for _ in range(q):
            qy, _ = qr_plus(y)
            z, _ = qr_plus(xn.T @ qy)
            y = xn @ z
    return y0, y


def khatri_rao(mats: Sequence[np.ndarray]) -> np.ndarray:
    """Column-wise Kronecker product A_1 (.) A_2 (.) ... (Eq. KHM): column c is
    kron(A_1[:, c], A_2[:, c], ...)."""
    k = mats[0].shape[1]
    out = np.ones((1, k))
    for m in mats:
        out = np.einsum("ic,jc->ijc", out, np.asarray(m, dtype=np.float64)).reshape(-1, k)
    return out


def sketch_kr(x: np.ndarray, n: int, omegas: Sequence[Optional[np.ndarray]], q: int = 0):
    """Khatri-Rao-structured mode-n sketch (P:510 footnote):
    Y0 = X_(n) (Omega_N (.) ... (.) Omega_1, without n), every Omega_k in R^{I_k x K}, in the
    Kronecker ordering of Eq.(2) so that the j-index of the unfolding matches.
    Power iterations (q > 0) continue with dense Z as in ``sketch_gauss``."""
    x64 = np.asarray(x, dtype=np.float64)
    xn = unfold(x64, n)
    kr = khatri_rao([omegas[k] for k in reversed(range(x64.ndim)) if k != n])
    y0 = xn @ kr
    y = y0
    for _ in range(q):
        qy, _ = qr_plus(y)
        z, _ = qr_plus(xn.T @ qy)
        y = xn @ z
    return y0, y


def count_decode(codes):
    """Split the caller-drawn codes code_j = s_j (h_j + 1) into the hash labels h_j in [0, K)
    and the Rademacher signs s_j (include/rtucker.h)."""
    c = np.asarray(codes, dtype=np.int64)
    if np.any(c == 0):
        raise ValueError("count-sketch code 0 is invalid")
    return np.abs(c) - 1, np.sign(c).astype(np.float64)


def sketch_count(x: np.ndarray, n: int, omega, q: int = 0):
    """Count-sketch mode-n sketch, the paper's three steps
    on the columns of X_(n): (1) hashing -- column j carries the label h_j in 1..K (here 0..K-1);
    (2) grouping the columns with the same label; (3) signing (s_j = +-1, footnote P:309) and
    summing each group into its representative column Y0[:, c].  omega = (codes, K).
    Power iterations (q > 0) continue with dense Z as in ``sketch_gauss``."""
    codes, K = omega
    xn = unfold(np.asarray(x, dtype=np.float64), n)
    h, s = count_decode(codes)
    if h.shape[0] != xn.shape[1] or np.any(h >= K):
        raise ValueError("count-sketch codes do not match the unfolding")
    y0 = np.zeros((xn.shape[0], K))
    for c in range(K):
        group = np.nonzero(h == c)[0]                       # step 2
        y0[:, c] = xn[:, group] @ s[group]                  # step 3: signed column sum
    y = y0
    for _ in range(q):
        qy, _ = qr_plus(y)
        z, _ = qr_plus(xn.T @ qy)
        y = xn @ z
    return y0, y


def sketch(x, n, kind, omega, q=0):
    if kind == "gauss":
        return sketch_gauss(x, n, omega, q)
    if kind == "kron":
        return sketch_kron(x, n, omega, q)
    if kind == "kr":
        return sketch_kr(x, n, omega, q)
    if kind == "count":
        return sketch_count(x, n, omega, q)
    raise ValueError(kind)


# ------------------------------------------------------------------------- core
def core(x: np.ndarray, qs: Sequence[np.ndarray]) -> np.ndarray:
    """G = X x_1 Q_1^T x_2 ... x_N Q_N^T in ascending mode order (Eq. Core)."""
    return multi_ttm(np.asarray(x, dtype=np.float64), [np.asarray(qm, dtype=np.float64) for qm in qs],
                     transpose=True)


def rel_error(x: np.ndarray, g: np.ndarray, qs: Sequence[np.ndarray]) -> float:
    """E = ||X - G x_1 Q_1 ... x_N Q_N||_F / ||X||_F by explicit reconstruction
    (Eq. Relativeerror; reading R12).  0 for an all-zero X (reading R7)."""
    x64 = np.asarray(x, dtype=np.float64)
    nx = fro(x64)
    if nx == 0.0:
        return 0.0
    return fro(x64 - reconstruct(g, qs)) / nx


def rel_error_gram(x: np.ndarray, g: np.ndarray) -> float:
    """Pythagorean diagnostic E_gram = sqrt(max(0, 1 - ||G||^2/||X||^2))."""
    nx = fro(x)
    if nx == 0.0:
        return 0.0
    return float(np.sqrt(max(0.0, 1.0 - (fro(g) / nx) ** 2)))


# ------------------------------------------------------------------- truncation
def eig_desc(m: np.ndarray):
    """Symmetric EVD with eigenvalues in descending order (Gram-EVD; R5)."""
    w, v = np.linalg.eigh(np.asarray(m, dtype=np.float64))
    idx = np.argsort(-w, kind="stable")
    return w[idx], v[:, idx]


def canon_sign(qn: np.ndarray, u: np.ndarray):
    """Reading R5: make the largest-|.| entry of each lifted column positive
    (lowest row on ties); apply the same flip to the small matrix u."""
    qn = qn.copy()
    u = u.copy()
    for r in range(qn.shape[1]):
        i = int(np.argmax(np.abs(qn[:, r])))      # first maximum = lowest row
        if qn[i, r] < 0:
            qn[:, r] = -qn[:, r]
            u[:, r] = -u[:, r]
    return qn, u


def truncate_hosvd(gt: np.ndarray, qts: Sequence[np.ndarray], ranks: Sequence[int]):
    """Reading R1 (a6): truncate the oversampled core G~ (K_1..K_N) to R_n by a small
    HOSVD: M_n = G~_(n) G~_(n)^T, U_n = top-R_n eigenvectors, Q_n = Q~_n U_n,
    G = G~ x_n U_n^T for all n."""
    us, qs = [], []
    for n, qt in enumerate(qts):
        gn = unfold(gt, n)
        _, v = eig_desc(gn @ gn.T)
        u = v[:, :ranks[n]]
        qn, u = canon_sign(qt @ u, u)
        us.append(u)
        qs.append(qn)
    g = multi_ttm(gt, us, transpose=True)
    return g, qs


# ----------------------------------------------------------------- drivers
def _zero_result(dims, ranks):
    qs = [np.eye(d, r) for d, r in zip(dims, ranks)]
    return dict(Q=qs, G=np.zeros(tuple(ranks)), E=0.0, E_gram=0.0, Y0=None, Qt=qs)


def hosvd(x: np.ndarray, ranks: Sequence[int], omegas, q: int = 0, kind: str = "gauss",
          with_error: bool = True) -> dict:
    """Randomized HOSVD = Alg.6 RP-HOSVD with oversampling / power
    iteration of Alg.1 and the R1 truncation.

    omegas[n]: Gaussian J_n x K_n (kind="gauss") or the per-mode list of
    Kronecker factors (kind="kron").  Every mode sketches X itself (Z = X is never
    updated, reading R9).
    """
    x64 = np.asarray(x, dtype=np.float64)
    if fro(x64) == 0.0:
        return _zero_result(x64.shape, ranks)
    y0s, qts = [], []
    for n in range(x64.ndim):
        y0, y = sketch(x64, n, kind, omegas[n], q)
        qt, _ = qr_plus(y)
        y0s.append(y0)
        qts.append(qt)
    gt = core(x64, qts)
    g, qs = truncate_hosvd(gt, qts, ranks)
    out = dict(Q=qs, G=g, Qt=qts, Gt=gt, Y0=y0s)
    if with_error:
        out["E"] = rel_error(x64, g, qs)
        out["E_gram"] = rel_error_gram(x64, g)
    return out


def sthosvd(x: np.ndarray, ranks: Sequence[int], omegas, q: int = 0, kind: str = "gauss",
            mode_order: Optional[Sequence[int]] = None, with_error: bool = True) -> dict:
    """Randomized STHOSVD = Alg.8 R-STHOSVD (Alg.4).

    S = X (R8); for n in mode_order (ascending by default):
      Q~ = qr+(sketch(S, n))               (Alg.1 lines 1-3)
      B  = S x_n Q~^T                      (Alg.1 line 4)
      M  = B_(n) B_(n)^T, U = top-R_n eigenvectors (Gram-EVD of B)
      Q_n = Q~ U (sign canon R5);  S = B x_n U^T   (Alg.1 lines 5-7, ΛV^T shortcut P:424)
    G = S.  ``omegas[n]`` must be sized for the current S (gen.synth.sthosvd_dims_before).
    """
    x64 = np.asarray(x, dtype=np.float64)
    N = x64.ndim
    order = list(range(N)) if mode_order is None else list(mode_order)
    if fro(x64) == 0.0:
        return _zero_result(x64.shape, ranks)
    s = x64
    qs = [None] * N
    qts = [None] * N
    y0s = [None] * N
    for n in order:
        y0, y = sketch(s, n, kind, omegas[n], q)
        qt, _ = qr_plus(y)
        b = ttm(s, qt.T, n)
        bn = unfold(b, n)
        _, v = eig_desc(bn @ bn.T)
        u = v[:, :ranks[n]]
        qn, u = canon_sign(qt @ u, u)
        s = ttm(b, u.T, n)
        qs[n], qts[n], y0s[n] = qn, qt, y0
    out = dict(Q=qs, G=s, Qt=qts, Y0=y0s)
    if with_error:
        out["E"] = rel_error(x64, s, qs)
        out["E_gram"] = rel_error_gram(x64, s)
    return out


def pet(x: np.ndarray, ranks: Sequence[int], omegas, omega_tildes, with_error: bool = True) -> dict:
    """Alg.9 R-PET, the randomized pass-efficient Tucker algorithm:

      Y_n = X_(n) Omega_n                     (line 1; Omega_n: J_n x K_n)
      [Q^(n), ~] = QR(Y_n)                    (line 2; qr+ of reading R5)
      H = X x_1 Omega~_1 x_2 ... x_N Omega~_N (line 3; Omega~_n: S_n x I_n, R_n <= K_n <= S_n)
      S = H x_n (Omega~_n Q^(n))^dagger       (line 4; Moore-Penrose pseudo-inverse, numpy.linalg.pinv)
      truncate S, Q^(n) to (R_1..R_N)         (line 5; reading R1: the small HOSVD of S, as in hosvd)

    Every sketch of lines 1 and 3 reads X only (no product depends on another): one pass.
    """
    x64 = np.asarray(x, dtype=np.float64)
    if fro(x64) == 0.0:
        return _zero_result(x64.shape, ranks)
    N = x64.ndim
    y0s, qts = [], []
    for n in range(N):
        y0 = unfold(x64, n) @ np.asarray(omegas[n], dtype=np.float64)
        qt, _ = qr_plus(y0)
        y0s.append(y0)
        qts.append(qt)
    h = multi_ttm(x64, [np.asarray(o, dtype=np.float64) for o in omega_tildes])
    s = multi_ttm(h, [np.linalg.pinv(np.asarray(o, dtype=np.float64) @ qt) for o, qt in zip(omega_tildes, qts)])
    g, qs = truncate_hosvd(s, qts, ranks)
    out = dict(Q=qs, G=g, Qt=qts, Gt=s, H=h, Y0=y0s)
    if with_error:
        out["E"] = rel_error(x64, g, qs)
        out["E_gram"] = rel_error_gram(x64, g)
    return out


def rp_hooi(x: np.ndarray, ranks: Sequence[int], q_init: Sequence[np.ndarray], omegas, with_error: bool = True) -> dict:
    """Alg.7 RP-HOOI, len(omegas) sweeps (reading R24: the stopping criterion is a
    fixed sweep count; the Gaussian Omega^(n) of every sweep and mode are inputs):

      for each sweep, for n = 1..N:
        S = X x_{p != n} Q^(p)T                     (line 4, the latest factors)
        W^(n) = S_(n) Omega^(n),  Omega^(n) in R^{prod_{p!=n} R_p x R_n}   (line 5)
        Q^(n) = orthonormal basis of W^(n) (qr+)      (line 6)
      S = S x_N Q^(N)T                               (line 7: the core of the last factors)

    Q^(n) are then sign-canonicalized (reading R5) and the core is X x_n Q^(n)T of those factors.
    """
    x64 = np.asarray(x, dtype=np.float64)
    N = x64.ndim
    qs = [np.asarray(q, dtype=np.float64) for q in q_init]
    for sweep in omegas:
        for n in range(N):
            s = multi_ttm(x64, qs, transpose=True, skip=[n])
            w = unfold(s, n) @ np.asarray(sweep[n], dtype=np.float64)
            qs[n], _ = qr_plus(w)
    qs = [canon_sign(q, np.zeros((1, q.shape[1])))[0] for q in qs]
    g = core(x64, qs)
    out = dict(Q=qs, G=g)
    if with_error:
        out["E"] = rel_error(x64, g, qs)
        out["E_gram"] = rel_error_gram(x64, g)
    return out


# ------------------------------------------------------ deterministic references
def thosvd(x: np.ndarray, ranks: Sequence[int]) -> dict:
    """Deterministic truncated HOSVD via full SVD of each unfolding (Eq. UnfoldHOSVD
    P:378-382, Core P:383-385); signs canonicalized like R5."""
    x64 = np.asarray(x, dtype=np.float64)
    qs = []
    for n in range(x64.ndim):
        u, _, _ = np.linalg.svd(unfold(x64, n), full_matrices=False)
        qn, _ = canon_sign(u[:, :ranks[n]], np.zeros((1, ranks[n])))
        qs.append(qn)
    g = core(x64, qs)
    return dict(Q=qs, G=g, E=rel_error(x64, g, qs))


def sthosvd_det(x: np.ndarray, ranks: Sequence[int], mode_order=None) -> dict:
    """Deterministic STHOSVD (Alg.4) via full SVD of S_(n)."""
    x64 = np.asarray(x, dtype=np.float64)
    order = list(range(x64.ndim)) if mode_order is None else list(mode_order)
    s = x64
    qs = [None] * x64.ndim
    for n in order:
        u, _, _ = np.linalg.svd(unfold(s, n), full_matrices=False)
        qn, _ = canon_sign(u[:, :ranks[n]], np.zeros((1, ranks[n])))
        qs[n] = qn
        s = ttm(s, qn.T, n)
    return dict(Q=qs, G=s, E=rel_error(x64, s, qs))


def hooi(x: np.ndarray, ranks: Sequence[int], iters: int = 50) -> dict:
    """Deterministic HOOI (Alg.5), THOSVD-initialized; used only by the
    quasi-optimality pin."""
    x64 = np.asarray(x, dtype=np.float64)
    qs = thosvd(x64, ranks)["Q"]
    for _ in range(iters):
        for n in range(x64.ndim):
            y = multi_ttm(x64, qs, transpose=True, skip=[n])
            u, _, _ = np.linalg.svd(unfold(y, n), full_matrices=False)
            qs[n] = u[:, :ranks[n]]
    g = core(x64, qs)
    return dict(Q=qs, G=g, E=rel_error(x64, g, qs))


__all__ = ["qr_plus", "sketch_gauss", "sketch_kron", "sketch_kr", "sketch_count", "count_decode", "khatri_rao", "sketch", "core", "rel_error", "pet",
           "rp_hooi",
           "rel_error_gram", "eig_desc", "canon_sign", "truncate_hosvd", "hosvd", "sthosvd",
           "thosvd", "sthosvd_det", "hooi", "unfold", "fold", "ttm", "multi_ttm", "reconstruct", "fro"]
