"""Parity of the tcgen05 (3xTF32, TMEM, TMA) TTM kernels, forced with RT_OPT_TTM_IMPL = 2,
against the fp64 oracle.  Tolerances as in test_gpu_parity (BASELINE north_star 1e-5)."""
import dataclasses

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


def _handle(P, impl=2, omega_tf32=False):
    from paper_2001_07124_b200 import _lib as L
    h = P.Handle()
    h.set_option(L.RT_OPT_TTM_IMPL, impl)
    h.set_option(L.RT_OPT_OMEGA_TF32, int(omega_tf32))
    return h


@pytest.fixture(scope="module")
def htc(P):
    h = _handle(P, 2)
    yield h
    h.close()


def dev(x):
    return torch.from_numpy(synth.to_device_layout(x)).cuda()


def om_dev(om):
    return torch.from_numpy(np.ascontiguousarray(om)).cuda()


def mat(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("dims,K", [((128, 96, 64), 80), ((500, 500, 40), 30), ((256, 36, 20, 12), 16),
                                    ((1024, 200), 64), ((132, 68, 260), 128)])
def test_tc_sketch_parity(P, htc, dims, K):
    x = np.asfortranarray(np.random.default_rng(1).standard_normal(dims).astype(np.float32))
    X = dev(x)
    rng = np.random.default_rng(2)
    for n in range(len(dims)):
        J = x.size // dims[n]
        om = rng.standard_normal((J, K)).astype(np.float32)
        y = mat(P.rtucker_sketch(htc, X, n, om_dev(om)))
        y0, _ = oracle.sketch_gauss(x, n, om, 0)
        err = M.rel_fro(y, y0)
        assert err <= 1e-5, (n, err)
    htc.sync()


def test_tc_sketch_tf32_exact_omega(P):
    """RT_OPT_OMEGA_TF32: with a host-rounded (tf32-exact) Omega the 2-product path is exact to fp32."""
    h = _handle(P, 2, omega_tf32=True)
    dims = (256, 128, 96)
    x = np.asfortranarray(np.random.default_rng(3).standard_normal(dims).astype(np.float32))
    X = dev(x)
    for n in range(3):
        om = synth.round_tf32(np.random.default_rng(4 + n).standard_normal((x.size // dims[n], 80)))
        y = mat(P.rtucker_sketch(h, X, n, om_dev(om)))
        y0, _ = oracle.sketch_gauss(x, n, om, 0)
        assert M.rel_fro(y, y0) <= 1e-5
    h.sync()
    h.close()


def test_tc_long_contraction_precision(P, htc):
    """Accumulation precision over a long contraction (J = 2^20): the TMEM fp32 accumulator is
    drained every 128 contraction elements into fp32 registers, split-K partials reduced in fp64
    (measured on B200: draining every 1024 elements gave 7.5e-6, never draining 2.6e-5)."""
    dims = (256, 1024, 1024)
    x = np.asfortranarray(np.random.default_rng(5).standard_normal(dims).astype(np.float32))
    X = dev(x)
    for n in (0, 2):
        J = x.size // dims[n]
        om = np.random.default_rng(6).standard_normal((J, 80)).astype(np.float32)
        y = mat(P.rtucker_sketch(htc, X, n, om_dev(om)))
        y0 = oracle.unfold(x.astype(np.float64), n) @ om.astype(np.float64)
        err = M.rel_fro(y, y0)
        print(f"mode {n}: long-contraction rel err {err:.3e}")
        assert err <= 2e-6
    htc.sync()


def test_tc_long_contraction_core(P, htc):
    """ttm_t (first core stage) over a 2048-long contraction: segmented TMEM accumulation."""
    dims, C = (2048, 128, 96), (80, 16, 16)
    x = np.asfortranarray(np.random.default_rng(9).standard_normal(dims).astype(np.float32))
    rng = np.random.default_rng(10)
    qs = [np.linalg.qr(rng.standard_normal((d, c)))[0] for d, c in zip(dims, C)]
    G, _ = P.rtucker_core(htc, dev(x), [torch.from_numpy(q).cuda() for q in qs], with_error=False)
    htc.sync()
    err = M.rel_fro(P.core_to_numpy(G), oracle.core(x, qs))
    print(f"core long-contraction rel err {err:.3e}")
    assert err <= 5e-6


@pytest.mark.parametrize("q", [1, 2])
def test_tc_power_iteration(P, htc, q):
    cfg = synth.CONFIGS["cfg2"].scaled((128, 100, 84), (8, 8, 8), (8, 8, 8))
    x = synth.make_tensor(cfg)
    X = dev(x)
    for n in range(3):
        om = synth.gaussian_omega(cfg, n, K=16)
        y = mat(P.rtucker_sketch(htc, X, n, om_dev(om), q=q))
        _, yo = oracle.sketch_gauss(x, n, om, q)
        ug = np.linalg.svd(y, full_matrices=False)[0][:, :8]
        uo = np.linalg.svd(yo, full_matrices=False)[0][:, :8]
        assert M.subspace(ug, uo) <= 1e-5
    htc.sync()


@pytest.mark.parametrize("scale", [1.0, 3e-12, 1e12])
@pytest.mark.parametrize("h16", [True, False])
def test_tc_power_iteration_h16(P, scale, h16):
    """The power product on the fp16-split kernel (ttm_s_h16, X scaled by a power of two taken from
    max|X|) against the 3xTF32 kernel and the oracle, at data scales far outside the fp16 range;
    ragged shapes, several K (tc_npad 16 .. 128)."""
    from paper_2001_07124_b200 import _lib as L
    h = _handle(P, 2, omega_tf32=True)
    h.set_option(L.RT_OPT_TC_ABLATE, 211 if h16 else 210)
    try:
        for dims, K in [((130, 100, 84), 16), ((256, 150, 70), 20), ((96, 140, 200), 48), ((140, 130, 150), 80),
                        ((200, 160, 130), 128)]:
            x = np.asfortranarray((np.random.default_rng(9).standard_normal(dims) * scale).astype(np.float32))
            X = dev(x)
            rng = np.random.default_rng(10)
            for n in range(3):
                om = synth.round_tf32(rng.standard_normal((x.size // dims[n], K)).astype(np.float32))
                y = mat(P.rtucker_sketch(h, X, n, om_dev(om), q=1))
                _, yo = oracle.sketch_gauss(x, n, om, 1)
                assert np.all(np.isfinite(y))
                # span(Y) = span(X_(n) X_(n)^T Q_y) does not depend on R_z (nor on its shift)
                sub = M.subspace(np.linalg.qr(y)[0], np.linalg.qr(yo)[0])
                assert sub <= 1e-5, (dims, K, n, sub)
        h.sync()
    finally:
        h.close()


@pytest.mark.parametrize("dims,C", [((128, 96, 64), (80, 16, 32)), ((500, 500, 40), (30, 30, 20))])
def test_tc_core_parity(P, htc, dims, C):
    x = np.asfortranarray(np.random.default_rng(7).standard_normal(dims).astype(np.float32))
    rng = np.random.default_rng(8)
    qs = [np.linalg.qr(rng.standard_normal((d, c)))[0] for d, c in zip(dims, C)]
    G, err = P.rtucker_core(htc, dev(x), [torch.from_numpy(q).cuda() for q in qs])
    htc.sync()
    go = oracle.core(x, qs)
    assert M.rel_fro(P.core_to_numpy(G), go) <= 1e-5
    assert abs(mat(err)[0] - oracle.rel_error(x, go, qs)) / oracle.rel_error(x, go, qs) <= 1e-5


@pytest.mark.parametrize("name,dims,core,ranks", [
    ("cfg5", (160, 152, 144), (40, 40, 40), (40, 40, 40)),
    ("cfg4", (320, 288, 64), (100, 100, 50), (30, 30, 12)),
    ("cfg2", (200, 180, 160), (20, 20, 20), (20, 20, 20)),
])
def test_tc_hosvd_parity(P, htc, name, dims, core, ranks):
    cfg = synth.CONFIGS[name].scaled(dims, core, ranks)
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=cfg.q)
    htc.set_option(1, 1)                      # RT_OPT_PROFILE: check the tcgen05 kernels ran
    res = P.rtucker_hosvd(htc, dev(x), cfg.ranks, cfg.p, cfg.q, [om_dev(o) for o in oms])
    htc.sync()
    htc.set_option(1, 0)
    names = {n for n, _, _ in htc.profile_read()[0]}
    # the X-streaming launches ran on the tensor cores: the sketches, the power products and the
    # first core stage (labels of csrc/pipeline.cu)
    assert "ttm_s_tc" in names and "core_first" in names, names
    assert cfg.q == 0 or ("ttm_t_tc_pow" in names and "ttm_s_tc_pow" in names), names
    qg = [mat(q) for q in res["Q"]]
    gg = P.core_to_numpy(res["G"])
    for n in range(3):
        assert M.orth(qg[n]) <= 1e-12
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5, (n, M.subspace(qg[n], ref["Q"][n]))
    assert M.core_in_oracle_basis(gg, qg, ref["G"], ref["Q"]) <= 1e-5
    assert M.recon(gg, qg, ref["G"], ref["Q"]) <= 1e-5
    e = mat(res["err"])[0]
    assert abs(e - ref["E"]) / ref["E"] <= 1e-5


@pytest.mark.parametrize("mode", [211, 212])
def test_tc_hosvd_h16_gate(P, mode):
    """R29's device-side gate: with the scale forced to 0 (option 212) every fp16-split launch stands
    down and its tf32 twin (launched beside it, gated on the same scale) produces the result --
    the same parity as the fp16 path (211) on the same inputs."""
    from paper_2001_07124_b200 import _lib as L
    h = _handle(P, 2, omega_tf32=True)
    h.set_option(L.RT_OPT_TC_ABLATE, mode)
    try:
        # K = R + p = 32 (a multiple of 4): the power products take the fp16 / twin kernels too
        cfg = synth.CONFIGS["cfg2"].scaled((200, 180, 160), (22, 22, 22), (22, 22, 22))
        x = synth.make_tensor(cfg)
        oms = [synth.round_tf32(synth.gaussian_omega(cfg, n)) for n in range(3)]
        ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
        res = P.rtucker_hosvd(h, dev(x), cfg.ranks, cfg.p, 1, [om_dev(o) for o in oms])
        h.sync()
        runs = _runs(h)
        if mode == 211:   # 3 Z = X^T Q_y + 3 Y = X Q_z + the first core stage, all fp16 split
            assert runs.get("h16_ran", 0) >= 7 and runs.get("tf32_twin_ran", 0) == 0, runs
        else:             # gate forced closed: every fp16 launch stood down, the twins did the work
            assert runs.get("h16_ran", 0) == 0 and runs.get("tf32_twin_ran", 0) >= 7, runs
        qg = [mat(q) for q in res["Q"]]
        gg = P.core_to_numpy(res["G"])
        for n in range(3):
            assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5, (mode, n, M.subspace(qg[n], ref["Q"][n]))
        assert M.core_in_oracle_basis(gg, qg, ref["G"], ref["Q"]) <= 1e-5
        assert M.recon(gg, qg, ref["G"], ref["Q"]) <= 1e-5
        e = mat(res["err"])[0]
        assert abs(e - ref["E"]) / ref["E"] <= 1e-5
    finally:
        h.close()


def _runs(h):
    """Device run counters of the gated fp16 / tf32-twin pairs since the last read (rt_profile_read)."""
    return {n: c for n, c, _ in h.profile_read()[0] if n in ("h16_ran", "tf32_twin_ran")}


@pytest.mark.parametrize("scale", [1e-31, 1e-28, 3e-12, 1.0, 1e12, 1e30])
def test_tc_hosvd_h16_scales(P, htc, scale):
    """HOSVD with q = 1 on the fp16-split kernels (power products Z = X^T Q_y, Y = X Q_z and the
    first core stage; X's scale gathered in the first sketch pass: the 'xscale' launch) at data
    scales far outside the fp16 range: parity with the oracle on the same scaled tensor.  K = R + p
    = 32 (a multiple of 4, so the power products take the fp16 kernels); the device run counters
    prove which kernel of each gated pair did the work: the fp16 split at every scale down to
    max|X| >= 2^-98 (1e-28: max|X| ~ 2e-29), the tf32 twins below (1e-31: max|X| ~ 2e-32, s 2^14
    would not be a finite fp32, R29).  The
    residual sums are taken at a power-of-two scale, so E holds at every scale."""
    cfg = synth.CONFIGS["cfg2"].scaled((200, 180, 160), (22, 22, 22), (22, 22, 22))
    assert cfg.ranks[0] + cfg.p == 32
    x = np.asfortranarray((synth.make_tensor(cfg).astype(np.float64) * scale).astype(np.float32))
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    _runs(htc)
    htc.set_option(1, 1)
    res = P.rtucker_hosvd(htc, dev(x), cfg.ranks, cfg.p, 1, [om_dev(o) for o in oms])
    htc.sync()
    htc.set_option(1, 0)
    prof = htc.profile_read()[0]
    names = {n for n, _, _ in prof}
    runs = {n: c for n, c, _ in prof if n in ("h16_ran", "tf32_twin_ran")}
    assert "xscale" in names and "absmax" not in names, names      # scale from the first pass, no extra pass
    if scale >= 1e-28:
        assert runs.get("h16_ran", 0) >= 7 and runs.get("tf32_twin_ran", 0) == 0, runs
    else:
        assert runs.get("h16_ran", 0) == 0 and runs.get("tf32_twin_ran", 0) >= 7, runs
    qg = [mat(q) for q in res["Q"]]
    gg = P.core_to_numpy(res["G"])
    for n in range(3):
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5, (n, M.subspace(qg[n], ref["Q"][n]))
    assert M.core_in_oracle_basis(gg, qg, ref["G"], ref["Q"]) <= 1e-5
    assert M.recon(gg, qg, ref["G"], ref["Q"]) <= 1e-5
    e = mat(res["err"])[0]
    assert abs(e - ref["E"]) / ref["E"] <= 1e-5


def test_tc_sthosvd_shrink(P, htc):
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"].scaled((96, 80, 64), (8, 8, 8), (8, 8, 8)), q=0)
    x = synth.make_tensor(cfg)
    d = list(cfg.dims)
    oms = []
    for n in range(3):
        J = int(np.prod([d[k] for k in range(3) if k != n]))
        oms.append(np.ascontiguousarray(synth.rng_for(77, 1, n).standard_normal((J, 16)).astype(np.float32)))
        d[n] = cfg.ranks[n]
    ref = oracle.sthosvd(x, cfg.ranks, oms, q=0)
    res = P.rtucker_sthosvd(htc, dev(x), cfg.ranks, 8, 0, [om_dev(o) for o in oms])
    htc.sync()
    qg = [mat(q) for q in res["Q"]]
    for n in range(3):
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
    assert abs(mat(res["err"])[0] - ref["E"]) / ref["E"] <= 1e-5


@pytest.mark.parametrize("dims,rank,p,q", [((512, 256, 48), 20, 12, 1),      # K = 32
                                           ((1024, 128, 40), 16, 8, 2),      # K = 24 (npad 32)
                                           ((512, 256, 16, 12), 8, 8, 1)])   # order 4
def test_fused_sketch1_core0(P, dims, rank, p, q):
    """The fused pass (sketch1_core0_kernel: the mode-1 Omega sketch and the first core stage
    X x_1 Q~_0^T from one read of X, 10 instead of 11 passes for a 3-way tensor) in bench.py's
    configuration (tf32-rounded Omega), on shapes it accepts (I_0 % 512 == 0, I_1 % 128 == 0): parity
    with the oracle, the fused launch seen in the profile, and the same result as the unfused path
    (option 290) to fp32 rounding."""
    from paper_2001_07124_b200 import _lib as L
    N = len(dims)
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled(dims, (rank,) * N, (rank,) * N), p=p, q=q)
    x = synth.make_tensor(cfg)
    oms = [synth.round_tf32(synth.gaussian_omega(cfg, n)) for n in range(N)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=q)
    res = {}
    for opt in (291, 290):
        h = _handle(P, 0, omega_tf32=True)
        h.set_option(L.RT_OPT_TC_ABLATE, opt)
        h.set_option(L.RT_OPT_PROFILE, 1)
        r = P.rtucker_hosvd(h, dev(x), cfg.ranks, cfg.p, q, [om_dev(o) for o in oms])
        h.sync()
        names = {n for n, _, _ in h.profile_read()[0]}
        assert ("sketch1_core0" in names) == (opt == 291), (opt, names)
        res[opt] = r
        qg = [mat(t) for t in r["Q"]]
        gg = P.core_to_numpy(r["G"])
        for n in range(N):
            assert M.orth(qg[n]) <= 1e-12
            assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5, (opt, n, M.subspace(qg[n], ref["Q"][n]))
        assert M.core_in_oracle_basis(gg, qg, ref["G"], ref["Q"]) <= 1e-5
        assert M.recon(gg, qg, ref["G"], ref["Q"]) <= 1e-5
        e = mat(r["err"])[0]
        assert abs(e - ref["E"]) / ref["E"] <= 1e-5, (opt, e, ref["E"])
        h.close()
    for n in range(N):
        assert M.subspace(mat(res[291]["Q"][n]), mat(res[290]["Q"][n])) <= 2e-6


@pytest.mark.parametrize("dims,rank", [((300, 200), 12), ((320, 256, 96), 12), ((2048, 96, 80), 10)])
def test_r31_unmix_steep_spectrum(P, dims, rank):
    """Reading R31': an R31 power step on Q_y unmixed by a sampled R_S (the default) against the QR of
    Z (option 240, the oracle's form) on spectra that fall steeply inside the sketch (sigma_1 / sigma_K
    ~ 400 for the order-2 case, which R31 without the unmixing missed at 1.07e-5): both within 2e-6
    of the oracle and of each other, with the fp16 power products seen running (device counters)."""
    from paper_2001_07124_b200 import _lib as L
    N = len(dims)
    cfg = dataclasses.replace(synth.CONFIGS["cfg2"].scaled(dims, (rank,) * N, (rank,) * N), q=1)
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(N)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    out = {}
    for opt in (241, 240):
        h = _handle(P, 0)
        h.set_option(L.RT_OPT_TC_ABLATE, opt)
        h.set_option(L.RT_OPT_PROFILE, 1)
        r = P.rtucker_hosvd(h, dev(x), cfg.ranks, cfg.p, 1, [om_dev(o) for o in oms])
        h.sync()
        prof = h.profile_read()[0]
        names = {n for n, _, _ in prof}
        runs = {n: c for n, c, _ in prof if n in ("h16_ran", "tf32_twin_ran")}
        assert ("zsample" in names) == (opt == 241), names
        assert runs.get("h16_ran", 0) >= N and runs.get("tf32_twin_ran", 0) == 0, runs
        out[opt] = [mat(q) for q in r["Q"]]
        for n in range(N):
            assert M.subspace(out[opt][n], ref["Q"][n]) <= 2e-6, (opt, n, M.subspace(out[opt][n], ref["Q"][n]))
        assert abs(mat(r["err"])[0] - ref["E"]) / ref["E"] <= 1e-5
        h.close()
    for n in range(N):
        assert M.subspace(out[241][n], out[240][n]) <= 2e-6


@pytest.mark.parametrize("rank,p", [(60, 12), (64, 16), (80, 16), (100, 12)])
def test_split_residual_widths(P, rank, p):
    """Reading R35 (the default HOSVD driver): E from the rank-K residual pass (fp16-split residual
    kernel at P-tile widths 96 / 128 for K = 72, 80, 96, 112) plus the truncated core energy, while
    the truncation runs on the side stream; against the oracle's E (1e-5) and against the rank-R
    residual after the truncation (option 296) to 1e-6."""
    from paper_2001_07124_b200 import _lib as L
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled((384, 320, 256), (rank,) * 3, (rank,) * 3), p=p, q=1)
    x = synth.make_tensor(cfg)
    oms = [synth.round_tf32(synth.gaussian_omega(cfg, n)) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    e = {}
    for opt in (297, 296):
        h = _handle(P, 0, omega_tf32=True)
        h.set_option(L.RT_OPT_TC_ABLATE, opt)
        h.set_option(L.RT_OPT_PROFILE, 1)
        r = P.rtucker_hosvd(h, dev(x), cfg.ranks, cfg.p, 1, [om_dev(o) for o in oms])
        h.sync()
        names = {n for n, _, _ in h.profile_read()[0]}
        assert "residual_tc" in names, names          # (K > 64: its SIMT twin is launched gated)
        e[opt] = float(mat(r["err"])[0])
        assert abs(e[opt] - ref["E"]) / ref["E"] <= 1e-5, (opt, e[opt], ref["E"])
        qg = [mat(q) for q in r["Q"]]
        for n in range(3):
            assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5
        h.close()
    assert abs(e[297] - e[296]) / e[296] <= 1e-6


@pytest.mark.parametrize("dims,rank,p", [((512, 256, 256), 20, 12),     # K = 32
                                         ((512, 384, 256), 64, 16),     # K = 80 (the bench width)
                                         ((1024, 128, 384), 40, 8)])    # K = 48
def test_two_fused_passes(P, dims, rank, p):
    """The 9-pass HOSVD schedule (N = 3, q = 1): [Z0 + S1] (the fused pass writing mode 0's power-step
    Z in the R31 fp16 form beside mode 1's Omega sketch) and [G1 + S2] (the first core stage beside
    the last mode's Omega sketch, X viewed with the last mode as rows).  Parity with the oracle, both
    fused launches seen in the profile, and the same result as the one-fusion schedule (option 298)
    to fp32 rounding."""
    from paper_2001_07124_b200 import _lib as L
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled(dims, (rank,) * 3, (rank,) * 3), p=p, q=1)
    x = synth.make_tensor(cfg)
    oms = [synth.round_tf32(synth.gaussian_omega(cfg, n)) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=1)
    res = {}
    for opt in (299, 298):
        h = _handle(P, 0, omega_tf32=True)
        h.set_option(L.RT_OPT_TC_ABLATE, opt)
        h.set_option(L.RT_OPT_PROFILE, 1)
        r = P.rtucker_hosvd(h, dev(x), cfg.ranks, cfg.p, 1, [om_dev(o) for o in oms])
        h.sync()
        prof = h.profile_read()[0]
        names = {n for n, _, _ in prof}
        if opt == 299:
            assert "sketch1_z0" in names and "sketch2_core0" in names, names
            runs = {n: c for n, c, _ in prof if n in ("h16_ran", "tf32_twin_ran")}
            assert runs.get("tf32_twin_ran", 0) == 0, runs
        else:
            assert "sketch1_core0" in names and "sketch1_z0" not in names, names
        res[opt] = r
        qg = [mat(t) for t in r["Q"]]
        gg = P.core_to_numpy(r["G"])
        for n in range(3):
            assert M.orth(qg[n]) <= 1e-12
            assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5, (opt, n, M.subspace(qg[n], ref["Q"][n]))
        assert M.core_in_oracle_basis(gg, qg, ref["G"], ref["Q"]) <= 1e-5
        assert M.recon(gg, qg, ref["G"], ref["Q"]) <= 1e-5
        e = mat(r["err"])[0]
        assert abs(e - ref["E"]) / ref["E"] <= 1e-5, (opt, e, ref["E"])
        h.close()
    for n in range(3):
        assert M.subspace(mat(res[299]["Q"][n]), mat(res[298]["Q"][n])) <= 2e-6
