"""Slab partitioning of the data-parallel path.

X is split along its LAST mode into contiguous slabs, one per rank.  With the paper's
first-mode-fastest unfolding (reading R6) the column index of X_(n) is
j = alpha + a*beta with beta running over the modes after n, whose slowest digit is the
last-mode index; a slab [lo, hi) of the last mode therefore owns the contiguous j-rows
[a_n*lo, a_n*hi) of Omega_n for every n < N-1 (a_n = prod_{k<N-1, k!=n} I_k), and the
rows [lo, hi) of the last factor.  Pure host logic: no arithmetic of the method.
"""
from typing import Optional, Sequence, Tuple


def slab_range(I_last: int, world: int, rank: int) -> Tuple[int, int]:
    """Balanced contiguous slab [lo, hi) of the last mode for `rank` of `world`
    (sizes differ by at most one; empty slabs when world > I_last)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    return rank * I_last // world, (rank + 1) * I_last // world


def omega_rows(dims: Sequence[int], n: int, lo: int, hi: int) -> Optional[Tuple[int, int]]:
    """(row0, rows) of the Gaussian test matrix Omega_n (J_n x K_n) that the rank owning the
    last-mode slab [lo, hi) holds; None for the last mode (Omega_{N-1} is replicated)."""
    N = len(dims)
    if not 0 <= n < N:
        raise ValueError(f"mode {n} out of range for order {N}")
    if n == N - 1:
        return None
    a = 1
    for k in range(N - 1):
        if k != n:
            a *= int(dims[k])
    return a * lo, a * (hi - lo)


def local_dims(dims: Sequence[int], lo: int, hi: int) -> list:
    """Dimensions of the local slab."""
    return list(dims[:-1]) + [hi - lo]
