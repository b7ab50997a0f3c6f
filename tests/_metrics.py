"""Parity metrics GPU vs oracle, numpy fp64 only."""
from __future__ import annotations

import numpy as np

import oracle


def rel_fro(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b.ravel())
    if nb == 0.0:
        return float(np.linalg.norm(a.ravel()))
    return float(np.linalg.norm((a - b).ravel()) / nb)


def subspace(qg, qo) -> float:
    """M2: ||Qg Qg^T - Qo Qo^T||_F / sqrt(R) computed with small matrices."""
    qg = np.asarray(qg, dtype=np.float64)
    qo = np.asarray(qo, dtype=np.float64)
    r = qo.shape[1]
    # ||A - B||^2 = ||A||^2 + ||B||^2 - 2 ||Qo^T Qg||^2 for orthogonal projectors A, B
    c = qo.T @ qg
    v = np.linalg.norm(qg.T @ qg) ** 2 + np.linalg.norm(qo.T @ qo) ** 2 - 2 * np.linalg.norm(c) ** 2
    return float(np.sqrt(max(v, 0.0)) / np.sqrt(r))


def aligned_cols(qg, qo) -> float:
    """M3: sign-aligned ||Qg - Qo||_F / ||Qo||_F."""
    s = np.sign(np.sum(qg * qo, axis=0))
    s[s == 0] = 1
    return rel_fro(qg * s, qo)


def core_in_oracle_basis(gg, qgs, go, qos) -> float:
    """M4: ||Gg x_n (Qo_n^T Qg_n) - Go|| / ||Go||."""
    t = np.asarray(gg, dtype=np.float64)
    for n, (qg, qo) in enumerate(zip(qgs, qos)):
        t = oracle.ttm(t, qo.T @ qg, n)
    return rel_fro(t, go)


def recon(gg, qgs, go, qos) -> float:
    """M5: ||[[Gg;Qg]] - [[Go;Qo]]|| / ||[[Go;Qo]]|| with small matrices only
    (orthonormal factors: ||[[G;Q]]|| = ||G||)."""
    t = np.asarray(gg, dtype=np.float64)
    for n, (qg, qo) in enumerate(zip(qgs, qos)):
        t = oracle.ttm(t, qo.T @ qg, n)
    a2 = np.linalg.norm(np.asarray(gg).ravel()) ** 2
    b2 = np.linalg.norm(np.asarray(go).ravel()) ** 2
    ab = float(np.sum(t * go))
    return float(np.sqrt(max(a2 + b2 - 2 * ab, 0.0)) / np.sqrt(b2)) if b2 > 0 else float(np.sqrt(a2))


def orth(q) -> float:
    """M7: ||Q^T Q - I||_F."""
    q = np.asarray(q, dtype=np.float64)
    return float(np.linalg.norm(q.T @ q - np.eye(q.shape[1])))


def min_rel_gap(m_unf) -> float:
    """Minimum relative consecutive gap of the top singular values (for asserting M3)."""
    s = np.linalg.svd(m_unf, compute_uv=False)
    return float(np.min(np.abs(np.diff(s))) / s[0]) if len(s) > 1 else 1.0
