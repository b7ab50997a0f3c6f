"""Oracle tensor algebra (fp64, numpy) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2001_07124_b200``) never imports it.

Tensors are numpy arrays indexed in math order X[i_1, ..., i_N] (0-based here,
1-based in the paper).
"""
from __future__ import annotations

import numpy as np


def unfold(x: np.ndarray, n: int) -> np.ndarray:
    """n-unfolding X_(n) in R^{I_n x prod_{k!=n} I_k}  (§II).

    X_(n)(i_n, j) = X(i_1..i_N) with j = sum_{k!=n} i_k J_k, J_k = prod_{m<k, m!=n} I_m
    (0-based form of the paper's j-index): the remaining modes are linearized
    first-mode-fastest, i.e. Fortran order after moving mode n to the front.
    """
    return np.reshape(np.moveaxis(x, n, 0), (x.shape[n], -1), order="F")


def fold(m: np.ndarray, n: int, shape) -> np.ndarray:
    """Inverse of ``unfold`` (fold(unfold(t,n),n) == t)."""
    shape = list(shape)
    moved = [shape[n]] + [s for k, s in enumerate(shape) if k != n]
    return np.moveaxis(np.reshape(m, moved, order="F"), 0, n)


def ttm(x: np.ndarray, b: np.ndarray, n: int) -> np.ndarray:
    """n-mode product X x_n B, B in R^{J x I_n}.

    (X x_n B)_{..j..} = sum_{i_n} x_{..i_n..} b_{j,i_n}   (the printed bound I_N
    is read as I_n).  Computed through the unfolding identity
    unfold(X x_n B, n) = B X_(n).
    """
    shape = list(x.shape)
    shape[n] = b.shape[0]
    return fold(b @ unfold(x, n), n, shape)


def multi_ttm(x: np.ndarray, mats, transpose: bool = False, skip=None) -> np.ndarray:
    """X x_1 M_1 x_2 ... x_N M_N in ascending mode order (Eq. Core P:383-385 with
    transpose=True gives X x_n M_n^T).  ``mats[n] is None`` or n in ``skip`` leaves mode n."""
    skip = set() if skip is None else set(skip)
    t = x
    for n, m in enumerate(mats):
        if m is None or n in skip:
            continue
        t = ttm(t, m.T if transpose else m, n)
    return t


def reconstruct(g: np.ndarray, factors) -> np.ndarray:
    """[[G; Q_1..Q_N]] = G x_1 Q_1 ... x_N Q_N  (Eq. HOSVD)."""
    return multi_ttm(g, factors)


def fro(x: np.ndarray) -> float:
    """Frobenius norm sqrt(sum x^2), read in memory order (no copy of a strided view)."""
    return float(np.linalg.norm(np.asarray(x, dtype=np.float64).ravel(order="K")))
