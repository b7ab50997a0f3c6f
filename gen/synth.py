"""Seeded synthetic inputs for the randomized Tucker/HOSVD hot path.

This module serves BOTH the fp64 oracle (``oracle/``) and the CUDA path
(``paper_2001_07124_b200``).  It holds none of the method's arithmetic: it only
draws random numbers and assembles the *input* tensors and the random test
matrices Omega that the method consumes (Omega is passed explicitly to both
sides, so neither side draws random numbers of its own).

Recipes (BASELINE.json configs):

  * low multilinear rank tensor  X_s = [[G; U_1, ..., U_N]]  with a Gaussian core
    and orthonormal factors (Q of a Gaussian matrix), §VIII "Random Low
    Multilinear Rank Tensors" (the paper's factors are Gaussian, the
    BASELINE configs ask for orthonormal ones);
  * noise  X = X_s + gamma*N,  gamma = rho*||X_s||_F / ||N||_F  with the realized
    ||N|| (PAPER.md Eq. noisytensor, SNR P:836-838; reading R11);
  * cfg4's decaying core  G_ijk = N(0,1) / (i*j*k), 1-based (reading R14);
  * Gaussian Omega_n in R^{J_n x K_n}, rows in the paper's j-index order
    (PAPER.md Eq. proj, j-index P:99-105), generated in fp64 and
    rounded to the working dtype (reading R15);
  * Kronecker Omega_k^{(n)} in R^{d_k x L_k} (reading R3).

Memory layout convention shared by both sides: a tensor with math shape
(I_1, ..., I_N) is stored first-mode-fastest.  In numpy that is
a Fortran-ordered array of shape (I_1..I_N); in torch it is a C-contiguous tensor
of shape (I_N..I_1) (``to_device_layout``).

Seeds: every random object draws from
``numpy.random.SeedSequence([BASE_SEED, cfg, object, mode, slab])``.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional, Sequence

import numpy as np

BASE_SEED = 2001_07124

# object ids inside the seed tuple
_OBJ_CORE, _OBJ_FACTOR, _OBJ_NOISE, _OBJ_OMEGA, _OBJ_KRON, _OBJ_OMEGA_TILDE, _OBJ_KR, _OBJ_HOOI = 1, 2, 3, 4, 5, 6, 7, 8
_OBJ_COUNT = 9


def rng_for(*key: int) -> np.random.Generator:
    """Deterministic PCG64 stream for a key tuple (cfg, object, mode, slab, ...)."""
    return np.random.default_rng(np.random.SeedSequence([BASE_SEED, *[int(k) for k in key]]))


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration (or a scaled-down variant of its recipe)."""
    name: str
    cfg_id: int
    dims: tuple
    dtype: str                      # "f64" | "f32"
    core_dims: tuple                # multilinear rank of the signal
    core_kind: str                  # "gauss" | "decay"
    noise: str                      # "abs" | "rel" | "none"
    noise_level: float
    ranks: tuple                    # target multilinear rank R_n
    p: int                          # oversampling
    q: int                          # power iterations
    algo: str                       # "hosvd" | "sthosvd"
    omega: str                      # "gauss" | "kron"

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == "f64" else np.float32

    @property
    def nbytes(self) -> int:
        return int(np.prod(self.dims)) * (8 if self.dtype == "f64" else 4)

    def J(self, n: int) -> int:
        return int(np.prod([d for k, d in enumerate(self.dims) if k != n]))

    def K(self, n: int) -> int:
        """Gaussian sketch width K_n = min(R_n + p, I_n, J_n) (reading R1)."""
        return min(self.ranks[n] + self.p, self.dims[n], self.J(n))

    def scaled(self, dims: Sequence[int], core_dims: Sequence[int], ranks: Sequence[int],
               name: Optional[str] = None) -> "Config":
        return dataclasses.replace(self, dims=tuple(dims), core_dims=tuple(core_dims),
                                   ranks=tuple(ranks), name=name or self.name + "-small")


# BASELINE.json configs[0..4]  (cfg1..cfg5)
CONFIGS = {
    "cfg1": Config("cfg1", 1, (64, 64, 64), "f64", (5, 5, 5), "gauss", "abs", 1e-6,
                   (5, 5, 5), 5, 0, "hosvd", "gauss"),
    "cfg2": Config("cfg2", 2, (500, 500, 500), "f32", (20, 20, 20), "gauss", "rel", 1e-2,
                   (20, 20, 20), 10, 1, "hosvd", "gauss"),
    "cfg3": Config("cfg3", 3, (128, 128, 128, 128), "f32", (16, 16, 16, 16), "gauss", "rel", 1e-3,
                   (16, 16, 16, 16), 8, 0, "sthosvd", "kron"),
    "cfg4": Config("cfg4", 4, (2048, 2048, 256), "f32", (200, 200, 100), "decay", "none", 0.0,
                   (50, 50, 20), 10, 2, "hosvd", "gauss"),
    "cfg5": Config("cfg5", 5, (2048, 2048, 2048), "f32", (64, 64, 64), "gauss", "rel", 1e-3,
                   (64, 64, 64), 16, 1, "hosvd", "gauss"),
}


def orthonormal_factor(rng: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    """Q factor of a Gaussian rows x cols matrix (BASELINE.json: "U_n orthonormal from QR")."""
    a = rng.standard_normal((rows, cols))
    qm, _ = np.linalg.qr(a)
    return qm


def make_core(cfg: Config) -> np.ndarray:
    """Signal core G (fp64, Fortran order)."""
    g = rng_for(cfg.cfg_id, _OBJ_CORE).standard_normal(cfg.core_dims)
    if cfg.core_kind == "decay":
        # reading R14: G_ijk = N(0,1) / (i*j*k) with 1-based indices
        for n, d in enumerate(cfg.core_dims):
            shape = [1] * cfg.order
            shape[n] = d
            g = g / np.arange(1, d + 1, dtype=np.float64).reshape(shape)
    return np.asfortranarray(g)


def make_factors(cfg: Config) -> list:
    return [orthonormal_factor(rng_for(cfg.cfg_id, _OBJ_FACTOR, n), cfg.dims[n], cfg.core_dims[n])
            for n in range(cfg.order)]


def _expand(core: np.ndarray, factors: Sequence[np.ndarray]) -> np.ndarray:
    """[[core; U_1..U_N]] by successive tensordot (input assembly only)."""
    t = core
    for n, u in enumerate(factors):
        # contract mode n of t with the columns of u, put the new axis back at n
        t = np.moveaxis(np.tensordot(u, t, axes=([1], [n])), 0, n)
    return np.asfortranarray(t)


def make_tensor(cfg: Config, return_parts: bool = False):
    """Host (numpy fp64 assembly, rounded to cfg dtype) input tensor X, Fortran order.

    Returns X in cfg dtype; with ``return_parts`` also (X_signal_fp64, core, factors, gamma).
    """
    core = make_core(cfg)
    factors = make_factors(cfg)
    xs = _expand(core, factors)
    gamma = 0.0
    x = xs
    if cfg.noise != "none":
        nz = np.asfortranarray(rng_for(cfg.cfg_id, _OBJ_NOISE).standard_normal(cfg.dims))
        if cfg.noise == "abs":
            gamma = cfg.noise_level
        else:  # reading R11: rho relative to ||X_s||_F with the realized ||N||_F
            gamma = cfg.noise_level * np.linalg.norm(xs.ravel(order="K")) / np.linalg.norm(nz.ravel(order="K"))
        x = np.asfortranarray(xs + gamma * nz)
    out = np.asfortranarray(x.astype(cfg.np_dtype))
    if return_parts:
        return out, xs, core, factors, gamma
    return out


def gaussian_omega(cfg: Config, n: int, K: Optional[int] = None, rows: Optional[int] = None,
                   row0: int = 0, tf32: bool = False) -> np.ndarray:
    """Gaussian Omega_n as a (J_n, K_n) array (element (j,k) = Omega_n(j,k)).

    ``rows``/``row0`` select a contiguous block of rows (a slab's local rows), drawn
    from the same stream as the full matrix so slabs and the whole agree bit-exactly.
    ``tf32``: round to tf32-exact values (``round_tf32``) before handing it to both sides.
    """
    K = cfg.K(n) if K is None else K
    J = cfg.J(n)
    rows = J - row0 if rows is None else rows
    rng = rng_for(cfg.cfg_id, _OBJ_OMEGA, n)
    if row0:
        rng.standard_normal(row0 * K)  # advance the stream (row-major draw order)
    om = rng.standard_normal((rows, K))
    if tf32 and cfg.dtype == "f32":
        return np.ascontiguousarray(round_tf32(om))
    return np.ascontiguousarray(om.astype(cfg.np_dtype))


def kr_omegas(cfg: Config, n: int, cur_dims: Sequence[int], K: Optional[int] = None) -> list:
    """Khatri-Rao factors of the mode-n sketch: Omega_k in R^{d_k x K_n} (row-major) for k != n,
    K_n = min(R_n + p, I_n, J_n) of the current sizes; None at k = n."""
    N = len(cur_dims)
    J = int(np.prod([cur_dims[k] for k in range(N) if k != n]))
    K = min(cfg.ranks[n] + cfg.p, cur_dims[n], J) if K is None else K
    return [None if k == n else np.ascontiguousarray(
        rng_for(cfg.cfg_id, _OBJ_KR, n, k).standard_normal((cur_dims[k], K)).astype(cfg.np_dtype))
        for k in range(N)]


def hooi_omegas(cfg: Config, sweeps: int) -> list:
    """RP-HOOI test matrices Omega^(n) in R^{prod_{p!=n} R_p x R_n} (fp64, row-major), per sweep."""
    N = cfg.order
    out = []
    for it in range(sweeps):
        row = []
        for n in range(N):
            rows = int(np.prod([cfg.ranks[p] for p in range(N) if p != n]))
            row.append(np.ascontiguousarray(rng_for(cfg.cfg_id, _OBJ_HOOI, it, n).standard_normal((rows, cfg.ranks[n]))))
        out.append(row)
    return out


def count_codes(cfg: Config, n: int, K: Optional[int] = None, J: Optional[int] = None, step: int = 0) -> tuple:
    """Count-sketch operand (codes, K) for mode n: label h_j uniform on [0, K) and
    Rademacher sign s_j per column j of the (J_n-column) unfolding, packed as the int32 code
    s_j (h_j + 1).  ``J`` defaults to J_n of X (STHOSVD passes the shrunken size, ``step`` keys
    the stream)."""
    K = cfg.K(n) if K is None else int(K)
    J = cfg.J(n) if J is None else int(J)
    rng = rng_for(cfg.cfg_id, _OBJ_COUNT, n, step)
    h = rng.integers(0, K, size=J, dtype=np.int64)
    s = rng.integers(0, 2, size=J, dtype=np.int64) * 2 - 1
    return (s * (h + 1)).astype(np.int32), K


def pet_sizes(cfg: Config, K: Optional[Sequence[int]] = None) -> tuple:
    """R-PET sketch sizes (Alg.9): K_n = min(R_n + p, I_n, J_n) and S_n = min(2 K_n + 1, I_n)."""
    ks = [cfg.K(n) for n in range(cfg.order)] if K is None else list(K)
    ss = [min(2 * k + 1, cfg.dims[n]) for n, k in enumerate(ks)]
    return ks, ss


def omega_tilde(cfg: Config, n: int, S: int) -> np.ndarray:
    """Gaussian Omega~_n in R^{S_n x I_n} of R-PET line 3, dtype of the tensor."""
    rng = rng_for(cfg.cfg_id, _OBJ_OMEGA_TILDE, n)
    return np.ascontiguousarray(rng.standard_normal((S, cfg.dims[n])).astype(cfg.np_dtype))


def round_tf32(a: np.ndarray) -> np.ndarray:
    """Round fp32/fp64 values to the nearest tf32 value (10-bit mantissa, ties to even), returned
    as float32.  Used to make Gaussian Omega tf32-exact BEFORE it is handed to both
    the oracle and the CUDA path, which then skips the A_hi * Omega_lo product."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(13)) & np.uint64(1)
    u = (u + np.uint64(0x0FFF) + lsb) & np.uint64(0xFFFFE000)
    return u.astype(np.uint32).view(np.float32).reshape(np.shape(a))


def kron_widths(cfg: Config, n: int) -> list:
    """Reading R3: uniform L = ceil((R_n+p)^(1/(N-1))) per other mode."""
    L = int(math.ceil((cfg.ranks[n] + cfg.p) ** (1.0 / (cfg.order - 1)) - 1e-12))
    return [L if k != n else 0 for k in range(cfg.order)]


def kron_omegas(cfg: Config, n: int, cur_dims: Sequence[int], widths: Optional[Sequence[int]] = None) -> list:
    """Kronecker sketch matrices Omega_k^{(n)} in R^{d_k x L_k} for k != n (None at k == n).

    ``cur_dims`` are the current mode sizes of the tensor being sketched (for
    STHOSVD, already-truncated modes have d_k = R_k).  C order (element (i,l) at i*L+l).
    """
    widths = kron_widths(cfg, n) if widths is None else widths
    out = []
    for k in range(cfg.order):
        if k == n:
            out.append(None)
            continue
        om = rng_for(cfg.cfg_id, _OBJ_KRON, n, k).standard_normal((cur_dims[k], widths[k]))
        out.append(np.ascontiguousarray(om.astype(cfg.np_dtype)))
    return out


def sthosvd_dims_before(cfg: Config, n: int, order: Optional[Sequence[int]] = None) -> list:
    """Mode sizes of the working tensor S when STHOSVD reaches mode n (Alg.8)."""
    order = list(range(cfg.order)) if order is None else list(order)
    d = list(cfg.dims)
    for m in order:
        if m == n:
            break
        d[m] = cfg.ranks[m]
    return d


def to_device_layout(x: np.ndarray):
    """Numpy (I_1..I_N) Fortran array -> C-contiguous view of shape (I_N..I_1) (same bytes)."""
    return np.ascontiguousarray(x.T)


def compression_inverse(dims: Sequence[int], ranks: Sequence[int]) -> float:
    """1/compression ratio S2/S1, S1 = prod I_n, S2 = prod R_n + sum I_n R_n."""
    s1 = float(np.prod([float(d) for d in dims]))
    s2 = float(np.prod([float(r) for r in ranks])) + float(sum(i * r for i, r in zip(dims, ranks)))
    return s2 / s1


# ---------------------------------------------------------------------------
# Device-side assembly (torch) for configurations too large for host fp64
# assembly (cfg5: 2048^3, 32 GiB fp32).  Same recipe; the random streams are
# torch's Philox (seeded per slab from the same key tuple), so the bytes differ
# from the numpy path -- such inputs are checked with sampled outputs and
# size-independent properties.
# ---------------------------------------------------------------------------

def _torch_seed(*key: int) -> int:
    return int(np.random.SeedSequence([BASE_SEED, *key]).generate_state(1, dtype=np.uint64)[0] & ((1 << 63) - 1))


def make_tensor_device(cfg: Config, device, slab_modes: int = 64, last_range: Optional[tuple] = None):
    """Assemble X on ``device`` (torch tensor of shape (I_N..I_1), cfg dtype).

    Core and factors come from the numpy streams (small); the expansion runs in
    fp64 slab by slab along the last mode; noise is torch Philox per slab with a
    two-pass realized-norm scaling (reading R11).  ``last_range=(lo, hi)`` builds
    only that slab of the last mode (multi-GPU: each rank builds its own slab).
    Returns (X, info) with info = dict(core, factors, gamma).
    """
    import torch
    core = make_core(cfg)
    factors = make_factors(cfg)
    N = cfg.order
    I_last = cfg.dims[-1]
    lo, hi = (0, I_last) if last_range is None else last_range
    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    dev = torch.device(device)
    g = torch.from_numpy(np.ascontiguousarray(core.T)).to(dev)          # shape (R_N..R_1)
    us = [torch.from_numpy(u).to(dev) for u in factors]
    # partial expansion over modes 0..N-2: W shape (R_N, I_{N-1}..I_1)
    w = g
    for n in range(N - 1):
        ax = N - 1 - n                                              # torch axis of math mode n
        w = torch.movedim(torch.tensordot(w, us[n], dims=([ax], [1])), -1, ax)
    lead = int(np.prod(cfg.dims[:-1]))
    w2 = w.reshape(w.shape[0], lead)                                # (R_N, J)
    x = torch.empty((hi - lo,) + tuple(reversed(cfg.dims[:-1])), dtype=tdt, device=dev)
    xf = x.view(hi - lo, lead)
    gamma = 0.0
    if cfg.noise == "rel":
        # ||X_s||_F = ||G||_F exactly for orthonormal factors; realized ||N|| needs pass 1
        nn2 = 0.0
        for s0 in range(0, I_last, slab_modes):
            s1 = min(I_last, s0 + slab_modes)
            gen = torch.Generator(device=dev).manual_seed(_torch_seed(cfg.cfg_id, _OBJ_NOISE, s0))
            nz = torch.randn((s1 - s0, lead), generator=gen, device=dev, dtype=torch.float64)
            nn2 += float((nz * nz).sum())
        gamma = cfg.noise_level * float(np.linalg.norm(core.ravel())) / math.sqrt(nn2)
    elif cfg.noise == "abs":
        gamma = cfg.noise_level
    u_last = us[-1]
    for s0 in range(0, I_last, slab_modes):
        s1 = min(I_last, s0 + slab_modes)
        a, b = max(s0, lo), min(s1, hi)
        if a >= b:
            continue
        blk = u_last[a:b] @ w2                                          # (b-a, J) fp64
        if cfg.noise != "none":
            gen = torch.Generator(device=dev).manual_seed(_torch_seed(cfg.cfg_id, _OBJ_NOISE, s0))
            nz = torch.randn((s1 - s0, lead), generator=gen, device=dev, dtype=torch.float64)
            blk += gamma * nz[a - s0:b - s0]
        xf[a - lo:b - lo] = blk.to(tdt)
    return x, dict(core=core, factors=factors, gamma=gamma)


def gaussian_omega_device(cfg: Config, n: int, device, K: Optional[int] = None,
                          row0: int = 0, rows: Optional[int] = None, chunk_rows: int = 1 << 20,
                          tf32: bool = False):
    """Gaussian Omega_n generated on device (torch Philox, seeded per 2^20-row chunk).

    Returned as a (rows, K_n) row-major tensor (the library's layout for test matrices).  Row blocks are drawn
    chunk-wise so that any contiguous row range (a slab's local rows) matches the full matrix
    bit-exactly.  ``tf32``: round to nearest tf32 (same rule as ``round_tf32``).
    """
    import torch
    K = cfg.K(n) if K is None else K
    J = cfg.J(n)
    rows = J - row0 if rows is None else rows
    tdt = torch.float64 if cfg.dtype == "f64" else torch.float32
    dev = torch.device(device)
    out = torch.empty((rows, K), dtype=tdt, device=dev)
    c0 = (row0 // chunk_rows) * chunk_rows
    for c in range(c0, row0 + rows, chunk_rows):
        gen = torch.Generator(device=dev).manual_seed(_torch_seed(cfg.cfg_id, _OBJ_OMEGA, n, c))
        blk = torch.randn((min(chunk_rows, J - c), K), generator=gen, device=dev, dtype=torch.float64)
        a, b = max(c, row0), min(c + blk.shape[0], row0 + rows)
        v = blk[a - c:b - c].to(tdt)
        if tf32 and tdt == torch.float32:
            u = v.view(torch.int32)
            u = (u + 0x0FFF + ((u >> 13) & 1)) & ~0x1FFF
            v = u.view(torch.float32)
        out[a - row0:b - row0] = v
    return out
