"""Multi-rank control flow of the slab-parallel path on CPU (gloo, world_size 2).

Each rank owns a last-mode slab (paper_2001_07124_b200.partition) and replays the exchange
sequence of DESIGN.md section 7 with oracle primitives and gloo collectives:
C1 allreduce of partial sketches / power products of modes n < N-1, C2 allreduce of the Gram
of the row-distributed tall matrices (CholeskyQR), C3 allreduce of Z = X_(N-1)^T Q, C4
allreduce of the core, C5 allreduce of the residual sums + allgather for the sign rule of the
last factor.  The result must equal the unsharded oracle (Alg.6 + reading R1), which pins the
partition math (Omega row ranges, slab offsets, which quantities are partial sums and which
are row-distributed) independently of the GPU.
"""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gen import synth
from oracle import rtucker as orc
from oracle.tensor import fro, multi_ttm, unfold
from paper_2001_07124_b200 import partition

DIMS = (12, 10, 9)          # last mode 9 over 2 ranks: uneven slabs 4 + 5
RANKS = (3, 3, 3)
P, Q = 2, 1


def _cfg():
    return dataclasses.replace(synth.CONFIGS["cfg2"].scaled(DIMS, RANKS, RANKS), p=P, q=Q)


def _allreduce(a: np.ndarray) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _allgather_rows(a: np.ndarray) -> np.ndarray:
    sizes = [None] * dist.get_world_size()
    dist.all_gather_object(sizes, a.shape[0])
    m = max(sizes)                                  # gloo gathers equal shapes: pad, then trim
    parts = [torch.zeros((m, a.shape[1]), dtype=torch.float64) for _ in sizes]
    mine = torch.zeros((m, a.shape[1]), dtype=torch.float64)
    mine[:a.shape[0]] = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_gather(parts, mine)
    return np.concatenate([p.numpy()[:s] for p, s in zip(parts, sizes)], axis=0)


def _cholqr_rows(y_local: np.ndarray) -> np.ndarray:
    """Q of a row-distributed tall matrix: Gram allreduce (C2) + Cholesky; R_ii > 0 so Q is
    the unique one of qr_plus for full column rank."""
    g = _allreduce(y_local.T @ y_local)
    r = np.linalg.cholesky(g).T
    return np.linalg.solve(r.T, y_local.T).T


def _worker(rank, world, port, cfg, x, omegas, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = x.ndim
        lo, hi = partition.slab_range(x.shape[-1], world, rank)
        xr = x[..., lo:hi]
        assert list(xr.shape) == partition.local_dims(x.shape, lo, hi)
        qts, y0s = [], []
        for n in range(N):
            xn = unfold(xr, n)
            if n < N - 1:
                row0, rows = partition.omega_rows(x.shape, n, lo, hi)
                om = omegas[n][row0:row0 + rows]
                y0 = _allreduce(xn @ om)                                    # C1
                y = y0
                for _ in range(cfg.q):
                    qy, _ = orc.qr_plus(y)                                   # replicated
                    z = _cholqr_rows(xn.T @ qy)                              # row-distributed Z, C2
                    y = _allreduce(xn @ z)                                   # C1
                qt, _ = orc.qr_plus(y)
            else:
                assert partition.omega_rows(x.shape, n, lo, hi) is None
                y0 = xn @ omegas[n]                                          # local rows [lo, hi)
                y = y0
                for _ in range(cfg.q):
                    qy = _cholqr_rows(y)                                     # C2
                    z, _ = orc.qr_plus(_allreduce(xn.T @ qy))                # C3, replicated
                    y = xn @ z
                qt = _cholqr_rows(y)                                         # rows [lo, hi) of Q~_{N-1}
                y0 = _allgather_rows(y0)
            y0s.append(y0)
            qts.append(qt)
        gt = _allreduce(multi_ttm(xr, qts, transpose=True))                   # C4
        # truncation (reading R1) runs redundantly; the sign rule of the last factor needs
        # its full column, gathered from the slabs (C5)
        us, qs = [], []
        for n in range(N):
            gn = unfold(gt, n)
            _, v = orc.eig_desc(gn @ gn.T)
            u = v[:, :cfg.ranks[n]]
            lifted = qts[n] @ u if n < N - 1 else _allgather_rows(qts[n] @ u)
            qn, u = orc.canon_sign(lifted, u)
            us.append(u)
            qs.append(qn if n < N - 1 else qn[lo:hi])
        g = multi_ttm(gt, us, transpose=True)
        sums = _allreduce(np.array([fro(xr - multi_ttm(g, qs)) ** 2, fro(xr) ** 2]))   # C5
        e = float(np.sqrt(sums[0] / sums[1]))
        ret[rank] = dict(y0=y0s, q=[qm for qm in qs[:-1]] + [_allgather_rows(qs[-1])], g=g, e=e, lo=lo, hi=hi)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_ranges():
    assert [partition.slab_range(9, 2, r) for r in range(2)] == [(0, 4), (4, 9)]
    assert [partition.slab_range(2048, 8, r)[0] for r in range(8)] == list(range(0, 2048, 256))
    assert partition.slab_range(1, 3, 0) == (0, 0)                  # empty slab allowed
    # j = alpha + a*beta: the slab's rows of X_(n) are contiguous and of the expected count
    x = np.arange(np.prod(DIMS), dtype=np.float64).reshape(DIMS, order="F")
    for n in range(2):
        row0, rows = partition.omega_rows(DIMS, n, 4, 9)
        np.testing.assert_array_equal(unfold(x, n)[:, row0:row0 + rows], unfold(x[..., 4:9], n))
    with pytest.raises(ValueError):
        partition.slab_range(4, 2, 2)


def test_slab_parallel_matches_unsharded_oracle():
    cfg = _cfg()
    x = np.asarray(synth.make_tensor(cfg), dtype=np.float64)
    omegas = [synth.gaussian_omega(cfg, n) for n in range(x.ndim)]
    ref = orc.hosvd(x, cfg.ranks, omegas, q=cfg.q)
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), cfg, x, omegas, ret), nprocs=2, join=True)
    assert sorted(ret.keys()) == [0, 1]
    assert (ret[0]["lo"], ret[0]["hi"], ret[1]["lo"], ret[1]["hi"]) == (0, 4, 4, 9)
    for r in range(2):
        out = ret[r]
        for n in range(x.ndim):
            np.testing.assert_allclose(out["y0"][n], ref["Y0"][n], rtol=0, atol=1e-12 * np.abs(ref["Y0"][n]).max())
            np.testing.assert_allclose(out["q"][n], ref["Q"][n], rtol=0, atol=1e-9)
        np.testing.assert_allclose(out["g"], ref["G"], rtol=0, atol=1e-9 * np.abs(ref["G"]).max())
        assert abs(out["e"] - ref["E"]) <= 1e-9 * ref["E"]


# ------------------------------------------------ slab-parallel R-STHOSVD (slab mode last)
def _sthosvd_worker(rank, world, port, ranks, x, omegas, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = x.ndim
        lo, hi = partition.slab_range(x.shape[-1], world, rank)
        s = x[..., lo:hi]
        qs = []
        for n in range(N):
            sn = unfold(s, n)
            if n < N - 1:
                a = int(np.prod([s.shape[k] for k in range(N - 1) if k != n]))
                y = _allreduce(sn @ omegas[n][a * lo:a * hi])               # C1 (slab's Omega rows)
                qt, _ = orc.qr_plus(y)
                b = orc.fold(qt.T @ sn, n, tuple(qt.shape[1] if k == n else s.shape[k] for k in range(N)))
                bn = unfold(b, n)
                m = _allreduce(bn @ bn.T)                                    # Gram of B_(n): partial sums
                _, v = orc.eig_desc(m)
                u = v[:, :ranks[n]]
                qn, u = orc.canon_sign(qt @ u, u)
                qs.append(qn)
            else:
                y = sn @ omegas[n]                                           # local rows of the slab mode
                qt = _cholqr_rows(y)                                         # C2
                b = _allreduce(qt.T @ sn)                                    # B = S x_{N-1} Q~^T (C4-like)
                _, v = orc.eig_desc(b @ b.T)
                u = v[:, :ranks[n]]
                lifted = _allgather_rows(qt @ u)
                qn, u = orc.canon_sign(lifted, u)
                qs.append(qn[lo:hi])
                b = orc.fold(b, n, tuple(b.shape[0] if k == n else s.shape[k] for k in range(N)))
            s = orc.ttm(b, u.T, n)
        sums = _allreduce(np.array([fro(x[..., lo:hi] - multi_ttm(s, qs)) ** 2, fro(x[..., lo:hi]) ** 2]))
        ret[rank] = dict(q=qs[:-1] + [_allgather_rows(qs[-1])], g=s, e=float(np.sqrt(sums[0] / sums[1])))
    finally:
        dist.destroy_process_group()


def test_slab_parallel_sthosvd_matches_unsharded_oracle():
    cfg = _cfg()
    x = np.asarray(synth.make_tensor(cfg), dtype=np.float64)
    rng = np.random.default_rng(90)
    omegas, d = [], list(x.shape)
    for n in range(x.ndim):
        J = int(np.prod(d)) // d[n]
        omegas.append(rng.standard_normal((J, min(cfg.ranks[n] + cfg.p, d[n], J))))
        d[n] = cfg.ranks[n]
    ref = orc.sthosvd(x, cfg.ranks, omegas, q=0)
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_sthosvd_worker, args=(2, _free_port(), cfg.ranks, x, omegas, ret), nprocs=2, join=True)
    for r in range(2):
        out = ret[r]
        for n in range(x.ndim):
            np.testing.assert_allclose(out["q"][n], ref["Q"][n], rtol=0, atol=1e-9)
        np.testing.assert_allclose(out["g"], ref["G"], rtol=0, atol=1e-9 * np.abs(ref["G"]).max())
        assert abs(out["e"] - ref["E"]) <= 1e-9 * ref["E"]
