"""Device-timed measurements of the SURVEY.md §8(f) rows beyond the bench path, on a BASELINE
config (default cfg5, X generated on the device): one JSON line per operation with the X-streaming
rate against the measured HBM copy peak (MEASURED_PEAKS.json).

    python tools/bench_rows.py [--cfg cfg5] [--reps 3]

Rows: count-sketch operator per mode (1 pass over X), Khatri-Rao sketch per mode (1 pass),
R-PET (N + 1 sketch passes + 1 residual pass), RP-HOOI one sweep (N passes + core + residual).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from gen import synth  # noqa: E402
from paper_2001_07124_b200 import api  # noqa: E402


def timed(h, fn, reps):
    fn()
    h.sync()
    best = None
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(h.stream)
        fn()
        e1.record(h.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    h.sync()
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="cfg5")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.cfg]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    h = api.Handle()
    h.set_option(3, 1)          # RT_OPT_OMEGA_TF32: test matrices are host-rounded to tf32 (R18), as in bench.py
    X, _ = synth.make_tensor_device(cfg, "cuda")
    xb = X.numel() * X.element_size()
    N = cfg.order

    # fp64 oracle timed beside each row on a bounded sample of the same recipe (host cores)
    import time
    import oracle
    scfg = cfg.scaled((192, 192, 192), (24, 24, 24), (24, 24, 24), name=cfg.name + "-sample")
    sx = synth.make_tensor(scfg)
    sxb = sx.size * 4

    def otime(fn):
        t0 = time.perf_counter()
        fn()
        return time.perf_counter() - t0

    def oracle_line(op, secs, passes):
        return {"value": passes * sxb / secs / 1e9, "unit": "GB/s", "kind": "oracle", "cores": len(os.sched_getaffinity(0)),
                "sample": f"{op} on 192^3 fp32, R=24 (same recipe), {secs:.2f} s"}

    def emit(op, ms, passes, extra=None, cpu=None):
        gbs = passes * xb / (ms * 1e-3) / 1e9
        line = {"op": op, "config": cfg.name, "ms": ms, "x_passes": passes, "x_GBps": gbs, "hbm_peak": peak,
                "frac": gbs / peak}
        line.update(extra or {})
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)

    cs_cpu = oracle_line("oracle.sketch(count) mode 0", otime(lambda: oracle.sketch(sx, 0, "count", synth.count_codes(scfg, 0))), 1)
    kr_cpu = oracle_line("oracle.sketch(kr) mode 0", otime(lambda: oracle.sketch(sx, 0, "kr", synth.kr_omegas(scfg, 0, scfg.dims))), 1)
    sks, sss = synth.pet_sizes(scfg)
    pet_cpu = oracle_line("oracle.pet", otime(lambda: oracle.pet(sx, scfg.ranks, [synth.gaussian_omega(scfg, n, K=sks[n]) for n in range(3)],
                                                                [synth.omega_tilde(scfg, n, sss[n]) for n in range(3)])), N + 2)
    q0s = oracle.hosvd(sx, scfg.ranks, [synth.gaussian_omega(scfg, n) for n in range(3)], q=0)["Q"]
    hooi_cpu = oracle_line("oracle.rp_hooi 1 sweep", otime(lambda: oracle.rp_hooi(sx, scfg.ranks, q0s, synth.hooi_omegas(scfg, 1))), N + 2)

    for n in range(N):
        codes, K = synth.count_codes(cfg, n)
        c = torch.from_numpy(codes).cuda()
        emit(f"count_sketch mode {n}", timed(h, lambda: api.rtucker_sketch(h, X, n, (c, K), kind="count"), a.reps), 1,
             {"K": K}, cs_cpu if n == 0 else None)
    for n in range(N):
        oms = [None if k == n else torch.from_numpy(synth.round_tf32(o)).cuda()
               for k, o in enumerate(synth.kr_omegas(cfg, n, cfg.dims))]
        K = cfg.K(n)
        emit(f"khatri_rao_sketch mode {n}", timed(h, lambda: api.rtucker_sketch(h, X, n, oms, kind="kr"), a.reps), 1,
             {"K": K}, kr_cpu if n == 0 else None)
    ks, ss = synth.pet_sizes(cfg)
    om = [torch.from_numpy(synth.round_tf32(synth.gaussian_omega(cfg, n, K=ks[n]))).cuda() for n in range(N)]
    omt = [torch.from_numpy(synth.round_tf32(synth.omega_tilde(cfg, n, ss[n]))).cuda() for n in range(N)]
    emit("r_pet", timed(h, lambda: api.rtucker_pet(h, X, cfg.ranks, om, omt), a.reps), N + 2,
         {"note": "N factor sketches + core sketch + residual pass"}, pet_cpu)
    del om, omt
    q0 = [torch.linalg.qr(torch.randn(d, r, dtype=torch.float64, device="cuda"))[0]
          for d, r in zip(cfg.dims, cfg.ranks)]
    hs = [[torch.from_numpy(o).cuda() for o in sw] for sw in synth.hooi_omegas(cfg, 1)]
    emit("rp_hooi 1 sweep", timed(h, lambda: api.rtucker_rp_hooi(h, X, cfg.ranks, q0, hs), a.reps), N + 2,
         {"note": "N S-chain passes (first stage on the tensor cores, R30) + core + residual"}, hooi_cpu)
    h.close()


if __name__ == "__main__":
    main()
