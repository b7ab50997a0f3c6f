"""Per-config measurement rows: every BASELINE.json configuration (cfg1..cfg5) through the C-ABI in
bench.py's launch configuration (tensor-core dispatch, tf32-rounded Gaussian Omega / Kronecker
factors, reading R18), device-timed with CUDA events on the handle's stream, with the algorithmic
bytes of SURVEY.md §8(d) against the measured HBM copy peak, and the fp64 oracle timed beside it on
the box's host cores (the whole config when it finishes in seconds, else a bounded sample of the
same recipe).  cfg4 runs both R-HOSVD and R-STHOSVD (the Table III pair).

    python tools/config_rows.py [--configs cfg1 cfg2 ...] [--reps 5] > profiles/r02_rows.jsonl

Bytes models (per call, excluding the residual pass that a8 reports apart):
  R-HOSVD, Gaussian: per mode (1 + 2q) passes over X plus the J_n x K_n test / power matrix each,
    plus the first core stage (X and its J_0 x K_0 output): bench.work_model.
  R-STHOSVD: per step the working tensor S_n is streamed by the sketch ((1 + 2q) passes; for the
    Kronecker chain, its first stage) and by the shrink B = S x_n Q~^T; S_0 = X (fp32), later S_n
    fp64 (reading R19): 2 (1 + q) |S_n| summed over the steps.
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402
from gen import synth  # noqa: E402
from paper_2001_07124_b200 import api as P  # noqa: E402


def dev_tensor(cfg):
    if cfg.nbytes > (1 << 30) + 1:
        return synth.make_tensor_device(cfg, "cuda")[0], None
    x = synth.make_tensor(cfg)
    return torch.from_numpy(synth.to_device_layout(x)).cuda(), x


def sthosvd_gauss_omegas(cfg, tf32=True, order=None):
    oms = []
    for n in range(cfg.order):
        d = synth.sthosvd_dims_before(cfg, n, order)
        J = int(np.prod([d[k] for k in range(cfg.order) if k != n]))
        o = synth.rng_for(cfg.cfg_id, 77, n).standard_normal((J, cfg.K(n)))
        oms.append(np.ascontiguousarray(synth.round_tf32(o) if tf32 else o.astype(np.float32)))
    return oms


def sthosvd_bytes(cfg, q):
    d = list(cfg.dims)
    tot = 0
    for n in range(cfg.order):
        esz = 4 if n == 0 else 8
        tot += 2 * (1 + q) * int(np.prod(d)) * esz
        d[n] = cfg.ranks[n]
    return tot


def timed(h, fn, reps):
    fn()
    h.sync()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(h.stream)
        r = fn()
        e1.record(h.stream)
        h.sync()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), r


def oracle_time(cfg, algo, budget_elems):
    """fp64 oracle on the config itself when small, else on a cube-ish sample of the same recipe."""
    c = cfg
    if int(np.prod(cfg.dims)) > budget_elems:
        side = int(round(budget_elems ** (1.0 / cfg.order)))
        c = cfg.scaled(tuple(min(side, d) for d in cfg.dims), tuple(min(side, r) for r in cfg.core_dims),
                       tuple(min(side // 2, r) for r in cfg.ranks), name=cfg.name + f"-sample{side}")
    x = synth.make_tensor(c)
    t0 = time.perf_counter()
    if algo == "hosvd":
        oracle.hosvd(x, c.ranks, [synth.gaussian_omega(c, n) for n in range(c.order)], q=c.q)
    elif c.omega == "kron":
        oracle.sthosvd(x, c.ranks, [synth.kron_omegas(c, n, synth.sthosvd_dims_before(c, n)) for n in range(c.order)],
                       q=c.q, kind="kron")
    else:
        oracle.sthosvd(x, c.ranks, sthosvd_gauss_omegas(c, tf32=False), q=c.q)
    secs = time.perf_counter() - t0
    nb = x.size * (8 if c.dtype == "f64" else 4)
    return {"value": nb / secs / 1e9, "unit": "GB/s of X", "kind": "oracle", "cores": len(os.sched_getaffinity(0)),
            "sample": f"oracle.{algo} on {'x'.join(map(str, c.dims))} ({c.name}), {secs:.2f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--oracle-elems", type=float, default=6.0e7)
    ap.add_argument("--profile", action="store_true", help="top kernel classes of each run to stderr")
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    for name in a.configs:
        cfg = synth.CONFIGS[name]
        X, _ = dev_tensor(cfg)
        h = P.Handle()
        h.set_option(3, 1)                       # RT_OPT_OMEGA_TF32 (test matrices tf32-rounded, R18)
        runs = []
        if cfg.algo == "hosvd":
            oms = [synth.gaussian_omega_device(cfg, n, "cuda", tf32=True) for n in range(cfg.order)]
            wm = bench.work_model(cfg)
            runs.append(("R-HOSVD (Alg.6)", "hosvd",
                         lambda: P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms),
                         wm["ttm_s"][0] + wm["ttm_t"][0]))
        if cfg.algo == "sthosvd" or name == "cfg4":
            if cfg.omega == "kron":
                ko = [[None if o is None else torch.from_numpy(np.ascontiguousarray(synth.round_tf32(o))).cuda()
                       for o in synth.kron_omegas(cfg, n, synth.sthosvd_dims_before(cfg, n))] for n in range(cfg.order)]
                runs.append(("R-STHOSVD (Alg.8), Kronecker sketch", "sthosvd",
                             lambda: P.rtucker_sthosvd(h, X, cfg.ranks, cfg.p, cfg.q, ko, kind="kron"),
                             sthosvd_bytes(cfg, 0)))
            else:
                go = [torch.from_numpy(o).cuda() for o in sthosvd_gauss_omegas(cfg)]
                runs.append(("R-STHOSVD (Alg.8), Gaussian sketch", "sthosvd",
                             lambda: P.rtucker_sthosvd(h, X, cfg.ranks, cfg.p, cfg.q, go),
                             sthosvd_bytes(cfg, cfg.q)))
        for label, algo, fn, nbytes in runs:
            ms, res = timed(h, fn, a.reps)
            # the residual pass (a8) timed apart: its kernels' device time in one profiled call
            h.profile_read()
            h.set_option(1, 1)
            fn()
            h.sync()
            h.set_option(1, 0)
            prof = sorted(h.profile_read()[0], key=lambda e: -e[2])
            if a.profile:
                print(f"[{name} {label}] " + ", ".join(f"{n}:{c}x {t:.3f}" for n, c, t in prof[:16]), file=sys.stderr,
                      flush=True)
            res_ms = sum(t for n, _, t in prof if n in bench.RESIDUAL_LABELS)
            pipe_ms = max(1e-6, ms - res_ms)
            # a fused pass reads X once for two contractions (DESIGN.md §6f / §6g): one |X| less each
            names = {n for n, _, _ in prof}
            nfused = sum(1 for f in ("sketch1_core0", "sketch1_z0", "sketch2_core0") if f in names)
            if algo == "hosvd":
                nbytes -= nfused * cfg.nbytes
            gbs = nbytes / (pipe_ms * 1e-3) / 1e9
            line = {"config": name, "op": label, "dims": list(cfg.dims), "dtype": cfg.dtype, "ranks": list(cfg.ranks),
                    "p": cfg.p, "q": cfg.q, "ms": ms, "residual_ms": res_ms, "pipeline_ms": pipe_ms,
                    "x_GB": cfg.nbytes / 1e9, "x_GBps": cfg.nbytes / (ms * 1e-3) / 1e9,
                    "bytes_model_GB": nbytes / 1e9, "fused_passes": nfused,
                    "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak},
                    "rel_err": float(res["err"][0]),
                    "cpu_baseline": oracle_time(cfg, algo, a.oracle_elems)}
            print(json.dumps(line), flush=True)
        h.close()
        del X
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
