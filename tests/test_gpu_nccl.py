"""The NCCL backend on a real GPU: a 1-rank NCCL communicator (ncclGetUniqueId / ncclCommInitRank
through the run-time loaded libnccl) with RT_OPT_FORCE_COLLECTIVES, so that every slab exchange of
the drivers (C1-C5 allreduces, the sign-candidate allgather, TSQR Grams) goes through ncclAllReduce /
ncclAllGather.  One rank: the results must equal the communicator-free run to rounding (and the oracle at 1e-5).
Several ranks cannot share one GPU under NCCL; the multi-rank exchanges are covered by the
loopback-communicator tests and the gloo replay (tests/test_dist_gloo.py)."""
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


def _dev(x):
    return torch.from_numpy(synth.to_device_layout(x)).cuda()


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_nccl_unique_id(P):
    uid = P.get_unique_id()
    assert len(uid) == 128 and any(uid)


@pytest.mark.parametrize("q", [0, 1])
def test_nccl_one_rank_hosvd_matches_plain_and_oracle(P, q):
    from paper_2001_07124_b200 import _lib as L
    import dataclasses
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"].scaled((96, 88, 80), (8, 8, 8), (8, 8, 8)), q=q)
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=q)
    hp = P.Handle()
    plain = P.rtucker_hosvd(hp, _dev(x), cfg.ranks, cfg.p, q, [_t(o) for o in oms])
    hp.sync()
    hn = P.Handle(nccl_id=P.get_unique_id(), nranks=1, rank=0)
    hn.set_option(L.RT_OPT_FORCE_COLLECTIVES, 1)
    res = P.rtucker_hosvd(hn, _dev(x), cfg.ranks, cfg.p, q, [_t(o) for o in oms], last_offset=0,
                          last_global=cfg.dims[2])
    hn.sync()
    for n in range(3):
        qa, qb = res["Q"][n].cpu().numpy(), plain["Q"][n].cpu().numpy()
        # q = 0: the same launches (metric floor ~1e-8, fp64 cancellation).  q = 1: the slab mode of a
        # distributed call takes the C3 form (fp32 partial Z, allreduce, then the fp16
        # [hi | lo] split) where the plain call splits the accumulator directly, and its QR is the
        # row-distributed one: two roundings of the same 22-bit product, ~1e-7 apart
        # (the slab mode of a thin slab, I_N(local) < 8 K, sketches with the tf32 3-product kernel where
        # the plain call uses the fp16 form of Omega: also two roundings of one product, ~3e-7 apart)
        assert M.subspace(qa, qb) <= (1e-7 if q == 0 and n < 2 else 1e-6), (n, M.subspace(qa, qb))
        assert M.subspace(qa, ref["Q"][n]) <= 1e-5
    assert abs(float(res["err"][0]) - ref["E"]) / ref["E"] <= 1e-5
    hn.close()
    hp.close()


def test_nccl_one_rank_sthosvd_and_count(P):
    from paper_2001_07124_b200 import _lib as L
    cfg = synth.CONFIGS["cfg2"].scaled((64, 60, 56), (6, 6, 6), (6, 6, 6))
    x = synth.make_tensor(cfg)
    hn = P.Handle(nccl_id=P.get_unique_id(), nranks=1, rank=0)
    hn.set_option(L.RT_OPT_FORCE_COLLECTIVES, 1)
    oms = [synth.count_codes(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1, kind="count")
    res = P.rtucker_hosvd(hn, _dev(x), cfg.ranks, cfg.p, 1, [(_t(c), k) for c, k in oms], kind="count",
                          last_offset=0, last_global=cfg.dims[2])
    hn.sync()
    for n in range(3):
        assert M.subspace(res["Q"][n].cpu().numpy(), ref["Q"][n]) <= 1e-5
    assert abs(float(res["err"][0]) - ref["E"]) / ref["E"] <= 1e-5
    kr = [synth.kron_omegas(cfg, n, synth.sthosvd_dims_before(cfg, n)) for n in range(3)]
    ref2 = oracle.sthosvd(x, cfg.ranks, kr, q=0, kind="kron")
    res2 = P.rtucker_sthosvd(hn, _dev(x), cfg.ranks, cfg.p, 0, [[None if o is None else _t(o) for o in row]
                                                                for row in kr], kind="kron",
                             last_offset=0, last_global=cfg.dims[2])
    hn.sync()
    for n in range(3):
        assert M.subspace(res2["Q"][n].cpu().numpy(), ref2["Q"][n]) <= 1e-5
    hn.close()
