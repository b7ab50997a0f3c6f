"""GPU parity of the count-sketch operator through the C-ABI
(kind "count") against the fp64 oracle on the same seeded codes.  Sketch: M1 relative Frobenius
<= 1e-5 (fp32 data, fp32 per-CTA partials of <= 512 terms combined in fp64) / 1e-12 (fp64);
drivers: M2, M4-M6 <= 1e-5, M7 <= 1e-12."""
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
    from paper_2001_07124_b200 import api
    return api


@pytest.fixture(scope="module")
def h(P):
    hh = P.Handle()
    yield hh
    hh.close()


def _dev(x):
    return torch.from_numpy(synth.to_device_layout(x)).cuda()


def _codes(rng, J, K):
    return ((rng.integers(0, K, J) + 1) * (2 * rng.integers(0, 2, J) - 1)).astype(np.int32)


def _c(codes):
    return torch.from_numpy(np.ascontiguousarray(codes)).cuda()


@pytest.mark.parametrize("dims,K,dtype", [
    ((37, 50, 29), 13, np.float32),          # ragged: partial row blocks and column blocks
    ((300, 260, 5), 40, np.float32),         # a = 300*260 for the last mode, tiny b
    ((20, 18, 16, 14), 9, np.float32),       # order 4
    ((700, 650), 100, np.float32),           # order 2, several row blocks (TI = 256)
    ((5, 7, 600), 5, np.float32),            # a = 5, 35: column blocks cross beta boundaries
    ((24, 22, 20), 11, np.float64),
    ((1, 40, 30), 1, np.float32),            # degenerate I_0 = 1, K = 1
])
def test_count_sketch_parity(P, h, dims, K, dtype):
    rng = np.random.default_rng(41)
    x = np.asfortranarray(rng.standard_normal(dims).astype(dtype))
    X = _dev(x)
    tol = 1e-5 if dtype == np.float32 else 1e-12
    for n in range(len(dims)):
        J = x.size // dims[n]
        k = min(K, J)
        codes = _codes(rng, J, k)
        y = P.rtucker_sketch(h, X, n, (_c(codes), k), kind="count").cpu().numpy()
        y0, _ = oracle.sketch(x, n, "count", (codes, k))
        assert M.rel_fro(y, y0) <= tol, (n, M.rel_fro(y, y0))
    h.sync()


def test_count_sketch_power_iteration(P, h):
    rng = np.random.default_rng(42)
    x = np.asfortranarray(rng.standard_normal((90, 80, 70)).astype(np.float32))
    codes = _codes(rng, 80 * 70, 12)
    y = P.rtucker_sketch(h, _dev(x), 0, (_c(codes), 12), q=1, kind="count").cpu().numpy()
    _, yq = oracle.sketch(x, 0, "count", (codes, 12), q=1)
    h.sync()
    assert M.subspace(np.linalg.qr(y)[0], np.linalg.qr(yq)[0]) <= 1e-5


def test_count_sketch_exact_integers(P, h):
    """Small-integer data: every partial sum is exact in fp32, so the sketch is bit-exact."""
    rng = np.random.default_rng(43)
    x = np.asfortranarray(rng.integers(-8, 9, (64, 48, 40)).astype(np.float32))
    X = _dev(x)
    for n in range(3):
        J = x.size // x.shape[n]
        codes = _codes(rng, J, 16)
        y = P.rtucker_sketch(h, X, n, (_c(codes), 16), kind="count").cpu().numpy()
        y0, _ = oracle.sketch(x, n, "count", (codes, 16))
        assert np.array_equal(y, y0), n
    h.sync()


@pytest.mark.parametrize("dims", [(2048, 96, 80), (96, 2048, 80), (64, 48, 4000)])
def test_count_sketch_bitwise_reproducible(P, h, dims):
    """Gaussian fp32 data (inexact partial sums): two calls give bit-identical sketches on every
    mode (per-CTA partial slices added in a fixed order, no floating-point atomics),
    across several CTAs per row block (each shape splits the columns over > 1 CTA)."""
    rng = np.random.default_rng(44)
    x = np.asfortranarray(rng.standard_normal(dims).astype(np.float32))
    X = _dev(x)
    for n in range(3):
        J = x.size // dims[n]
        codes = _c(_codes(rng, J, 24))
        ys = [P.rtucker_sketch(h, X, n, (codes, 24), kind="count").cpu().numpy() for _ in range(3)]
        assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[0], ys[2]), n
    h.sync()


@pytest.mark.parametrize("q", [0, 1])
def test_count_hosvd_parity(P, h, q):
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"].scaled((120, 110, 100), (10, 10, 10), (10, 10, 10)), q=q)
    x = synth.make_tensor(cfg)
    oms = [synth.count_codes(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=q, kind="count")
    res = P.rtucker_hosvd(h, _dev(x), cfg.ranks, cfg.p, q, [(_c(c), k) for c, k in oms], kind="count")
    h.sync()
    qg = [t.cpu().numpy() for t in res["Q"]]
    gg = P.core_to_numpy(res["G"])
    for n in range(3):
        assert M.orth(qg[n]) <= 1e-12
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert M.core_in_oracle_basis(gg, qg, ref["G"], ref["Q"]) <= 1e-5
    assert M.recon(gg, qg, ref["G"], ref["Q"]) <= 1e-5
    assert abs(float(res["err"][0]) - ref["E"]) / ref["E"] <= 1e-5


def test_count_hosvd_exact_rank_fp64(P, h):
    """Pin P31 on the GPU: exact multilinear rank, K = R + p -> E < 1e-10 (fp64 data)."""
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS["cfg1"].scaled((40, 36, 32), (4, 4, 4), (4, 4, 4)), noise="none")
    x = synth.make_tensor(cfg)
    oms = [synth.count_codes(cfg, n) for n in range(3)]
    res = P.rtucker_hosvd(h, _dev(x), cfg.ranks, cfg.p, 0, [(_c(c), k) for c, k in oms], kind="count")
    h.sync()
    assert float(res["err"][0]) < 1e-10


def test_count_sthosvd_parity(P, h):
    cfg = synth.CONFIGS["cfg3"].scaled((40, 36, 32, 30), (6, 6, 6, 6), (6, 6, 6, 6))
    x = synth.make_tensor(cfg)
    oms = []
    for n in range(4):
        d = synth.sthosvd_dims_before(cfg, n)
        J = math.prod(d) // d[n]
        oms.append(synth.count_codes(cfg, n, K=min(cfg.ranks[n] + cfg.p, d[n], J), J=J, step=1))
    ref = oracle.sthosvd(x, cfg.ranks, oms, q=0, kind="count")
    res = P.rtucker_sthosvd(h, _dev(x), cfg.ranks, cfg.p, 0, [(_c(c), k) for c, k in oms], kind="count")
    h.sync()
    qg = [t.cpu().numpy() for t in res["Q"]]
    for n in range(4):
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert abs(float(res["err"][0]) - ref["E"]) / ref["E"] <= 1e-5


def test_count_invalid_codes(P, h):
    from paper_2001_07124_b200 import _lib as L
    x = _dev(np.asfortranarray(np.ones((8, 9, 10), np.float32)))
    bad = np.full(90, 5, np.int32)                     # label 5 > K = 4: latched, reported by rt_sync
    P.rtucker_sketch(h, x, 0, (_c(bad), 4), kind="count")
    with pytest.raises(L.RtError):
        h.sync()
    h.sync()                                           # the latch is cleared
    with pytest.raises(ValueError):
        P.rtucker_sketch(h, x, 0, (_c(bad).to(torch.int64), 4), kind="count")
    with pytest.raises(L.RtError):                     # K > 128
        P.rtucker_sketch(h, x, 2, (_c(np.ones(72, np.int32)), 200), kind="count")
    h.sync()


def test_count_full_size_sampled_rows(P, h):
    """cfg5's size (2048^3 fp32, the bench tensor), K = 80: sampled sketch rows against fp64 sums
    of whole X_(n) rows computed one by one on the host (np.bincount of the signed row)."""
    cfg = synth.CONFIGS["cfg5"]
    X, _ = synth.make_tensor_device(cfg, "cuda")
    rng = np.random.default_rng(44)
    for n in range(3):
        codes, K = synth.count_codes(cfg, n)
        y = P.rtucker_sketch(h, X, n, (_c(codes), K), kind="count").cpu().numpy()
        hh, s = oracle.count_decode(codes)
        for i in rng.integers(0, cfg.dims[n], 3):
            # device layout (I_3, I_2, I_1): X_(n) row i in the Kolda j order, as fp64 on the host
            row = X.select(2 - n, int(i)).reshape(-1).double().cpu().numpy()
            ref = np.bincount(hh, weights=s * row, minlength=K)
            assert np.linalg.norm(y[i] - ref) <= 1e-5 * np.linalg.norm(ref), (n, i)
    h.sync()
    del X
    torch.cuda.empty_cache()


@pytest.mark.parametrize("nranks", [2, 3])
def test_count_loopback_multirank(P, nranks):
    """Slab-parallel count sketches: modes n < N-1 take the slab's block of codes (j = alpha +
    a beta) and allreduce (C1); the last mode's rows stay local with the full code array."""
    cfg = synth.CONFIGS["cfg5"].scaled((40, 36, 32), (5, 5, 5), (5, 5, 5))
    x = synth.make_tensor(cfg)
    oms = [synth.count_codes(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=cfg.q, kind="count")
    cuts = np.linspace(0, cfg.dims[2], nranks + 1).astype(int)
    grp = P.LoopbackGroup(nranks)
    out, errs = [None] * nranks, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                hh = P.Handle(stream=s, loopback_group=grp, rank=r)
                lo, hi = int(cuts[r]), int(cuts[r + 1])
                xs = _dev(np.asfortranarray(x[:, :, lo:hi]))
                a = [cfg.dims[1], cfg.dims[0]]
                loc = [(_c(oms[n][0][a[n] * lo:a[n] * hi]), oms[n][1]) for n in range(2)] + \
                      [(_c(oms[2][0]), oms[2][1])]
                res = P.rtucker_hosvd(hh, xs, cfg.ranks, cfg.p, cfg.q, loc, kind="count", last_offset=lo,
                                      last_global=cfg.dims[2])
                hh.sync()
                out[r] = dict(Q=[t.cpu().numpy() for t in res["Q"]], err=res["err"].cpu().numpy())
                hh.close()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not errs, errs
    qg = out[0]["Q"][:2] + [np.concatenate([out[r]["Q"][2] for r in range(nranks)], axis=0)]
    for n in range(3):
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert abs(out[0]["err"][0] - ref["E"]) / ref["E"] <= 1e-5
