"""Slab-wise evaluation of ``oracle.hosvd`` for tensors larger than the host RAM allows the plain
oracle (BASELINE.json cfg5: X = 2048^3, 69 GB in fp64; ``oracle.hosvd`` holds X, an explicit
unfolding and, for E, the full reconstruction and the difference: ~4 x 69 GB on a 196 GB host)
-- TEST INFRASTRUCTURE ONLY (``tests/`` may use it; the product path never imports it).

Same algorithm, same order of steps and the same oracle primitives (``unfold``, ``qr_plus``,
``core``, ``truncate_hosvd``, ``reconstruct``) as ``oracle.rtucker.hosvd`` with Gaussian test
matrices (Alg.6; Alg.1 lines 1-3 P:202-206 with the power iteration of reading R2;
truncation reading R1; E of Eq. Relativeerror).  The only change is that every sum
over the last mode is split into partial sums over contiguous slabs X[..., k0:k1] (a
reassociation of the same sums, SURVEY.md §8(c.4) pin P18; ``tests/test_oracle_pins.py`` pins
this module against ``oracle.hosvd``):

  * mode n < N-1: X_(n) = [X_(n)^(1) | X_(n)^(2) | ...] column blocks (the last mode is the
    slowest index of the paper's j-index), so X_(n) B = sum_s X_(n)^(s) B[rows_s] and
    X_(n)^T Q stacks the slab blocks;
  * mode N-1: X_(N-1) = row blocks, so X_(N-1) Z stacks and X_(N-1)^T Q = sum_s X_(N-1)^(s)T Q[k0:k1];
  * core: G~ = sum_s core(X^(s), [Q~_1, ..., Q~_N[k0:k1]]) (multilinear in the last factor);
  * E: ||X - X^||^2 = sum_s ||X^(s) - reconstruct(G, [Q_1, ..., Q_N[k0:k1]])||^2.
"""
from __future__ import annotations

import os
import sys
import time
from typing import Sequence

import numpy as np

from .rtucker import _zero_result, core, qr_plus, rel_error_gram, truncate_hosvd
from .tensor import fro, reconstruct, unfold


def _slabs(last: int, width: int):
    return [(k0, min(last, k0 + width)) for k0 in range(0, last, width)]


def hosvd_slabs(x: np.ndarray, ranks: Sequence[int], omegas, q: int = 0, slab: int = 64,
                with_error: bool = True) -> dict:
    """``oracle.hosvd(x, ranks, omegas, q)`` (Gaussian kind) evaluated slab by slab along the last
    mode.  ``x``: math order (I_1..I_N), any float dtype (each slab is widened to fp64; an
    F-ordered fp64 x is read through views).  Returns the same keys as ``oracle.hosvd``."""
    N = x.ndim
    dims = x.shape
    last = dims[-1]
    sl = _slabs(last, slab)
    # middle modes 0 < n < N-1: single-index slabs, whose unfolding of an F-ordered x is a strided
    # view (no copy of the slab per product); the first and last modes take the wide slabs
    sl1 = _slabs(last, 1)
    verbose = bool(os.environ.get("RT_ORACLE_VERBOSE"))
    t0 = time.perf_counter()

    def tick(what):
        if verbose:
            print(f"[hosvd_slabs] {what}: {time.perf_counter() - t0:.1f} s", file=sys.stderr, flush=True)

    def xs_of(k0, k1):
        return np.asarray(x[..., k0:k1], dtype=np.float64)

    def rows(n, k0, k1):
        # j-index rows of the slab in X_(n), n < N-1: the last mode is the slowest index
        jp = int(np.prod([dims[m] for m in range(N - 1) if m != n]))
        return slice(jp * k0, jp * k1)

    nx2 = sum(fro(xs_of(k0, k1)) ** 2 for k0, k1 in sl)
    if nx2 == 0.0:
        return _zero_result(dims, ranks)
    omegas = [np.asarray(o, dtype=np.float64) for o in omegas]

    def slabs_for(n):
        return sl1 if 0 < n < N - 1 else sl

    def x_times(n, b):                       # X_(n) B
        if n < N - 1:
            return sum(unfold(xs_of(k0, k1), n) @ b[rows(n, k0, k1)] for k0, k1 in slabs_for(n))
        return np.concatenate([unfold(xs_of(k0, k1), n) @ b for k0, k1 in sl], axis=0)

    def xt_times(n, qm):                     # X_(n)^T Q
        if n < N - 1:
            return np.concatenate([unfold(xs_of(k0, k1), n).T @ qm for k0, k1 in slabs_for(n)], axis=0)
        return sum(unfold(xs_of(k0, k1), n).T @ qm[k0:k1] for k0, k1 in sl)

    y0s, qts = [], []
    for n in range(N):
        # sketch_gauss (Alg.6 line 3, reading R2): Y0 = X_(n) Omega; q times Q = qr+(Y),
        # Z = qr+(X_(n)^T Q), Y = X_(n) Z
        y0 = x_times(n, omegas[n])
        y = y0
        for _ in range(q):
            qy, _ = qr_plus(y)
            z, _ = qr_plus(xt_times(n, qy))
            y = x_times(n, z)
        qt, _ = qr_plus(y)                   # Alg.6 line 4
        y0s.append(y0)
        qts.append(qt)
        tick(f"mode {n} sketch + {q} power iterations + QR")
    gt = sum(core(xs_of(k0, k1), qts[:-1] + [qts[-1][k0:k1]]) for k0, k1 in sl)   # line 5
    tick("core")
    g, qs = truncate_hosvd(gt, qts, ranks)                                        # reading R1
    out = dict(Q=qs, G=g, Qt=qts, Gt=gt, Y0=y0s)
    if with_error:
        res2 = sum(fro(xs_of(k0, k1) - reconstruct(g, qs[:-1] + [qs[-1][k0:k1]])) ** 2 for k0, k1 in sl)
        tick("residual")
        out["E"] = float(np.sqrt(res2 / nx2))
        out["E_gram"] = rel_error_gram(np.array([np.sqrt(nx2)]), g)   # only ||X|| enters the identity
    return out


__all__ = ["hosvd_slabs"]
