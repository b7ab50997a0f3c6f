"""Benchmark of the randomized Tucker/HOSVD hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl ours|reference]

A step = one rtucker_hosvd call (sketch + power iteration + thin QR + core + truncation +
relative error: every SURVEY.md §8(a) row of the HOSVD path) over the whole workload,
inputs resident in HBM.  N > 1: launched by torchrun, one rank per GPU, X sliced into slabs
along its last mode; partial sums are combined by NCCL inside librtucker.
Total work is fixed as N grows ("strong" scaling).  Time: CUDA events on the handle's
stream, barrier + synchronize on both sides, max over ranks.

--impl reference: the fp64 oracle (``oracle/``), as it stands, on the host cores on a
bounded sample of the same workload (rank 0 only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from gen import synth  # noqa: E402
from paper_2001_07124_b200 import partition  # noqa: E402

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
UNIT = "GB/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------- work model
def work_model(cfg, nranks=1, omega_products=2):
    """Algorithmic bytes / flops per rank per step, by kernel class.

    ttm_s (sketch & power products Y = X_(n) B): per launch reads X_local and B (J_n x K_n);
    flops 2 |X| K_n.  ttm_t (Z = X^T Q and the first core stage): reads X_local, writes
    J_n x K_n; flops 2 |X| K_n.  residual: reads X_local and P, flops 2 |X| R_N.
    """
    N = cfg.order
    esz = 8 if cfg.dtype == "f64" else 4
    dims = list(cfg.dims)
    dims_l = dims[:-1] + [dims[-1] // nranks]
    xl = int(np.prod(dims_l))
    K = [cfg.K(n) for n in range(N)]
    J_l = [xl // dims_l[n] for n in range(N)]
    s_bytes = s_flops = s_n = 0
    t_bytes = t_flops = t_n = 0
    for n in range(N):
        for _ in range(1 + cfg.q):
            s_bytes += xl * esz + J_l[n] * K[n] * esz
            s_flops += 2 * xl * K[n]
            s_n += 1
        for _ in range(cfg.q):
            t_bytes += xl * esz + J_l[n] * K[n] * esz
            t_flops += 2 * xl * K[n]
            t_n += 1
    # first core stage (mode 0): reads X, writes K_0 x J_0
    t_bytes += xl * esz + J_l[0] * K[0] * esz
    t_flops += 2 * xl * K[0]
    t_n += 1
    r_bytes = xl * esz + (xl // dims_l[-1]) * cfg.ranks[-1] * esz
    r_flops = 2 * xl * cfg.ranks[-1]
    total_flops = s_flops + t_flops + r_flops
    # hardware tensor flops of the ttm_s class: the Omega sketch runs 2 tf32 products (tf32-exact
    # Omega, reading R18); the power product Y = X Q_z runs 3 fp16 products (fp16 split, R29)
    s_hw_tf32 = sum(2 * xl * K[n] * omega_products for n in range(N))
    s_hw_f16 = sum(2 * xl * K[n] * 3 * cfg.q for n in range(N))
    return {"ttm_s": (s_bytes, s_flops, s_n), "ttm_t": (t_bytes, t_flops, t_n), "residual": (r_bytes, r_flops, 1),
            "total_flops": total_flops, "x_bytes_local": xl * esz, "ttm_s_hw_tf32": s_hw_tf32,
            "ttm_s_hw_f16": s_hw_f16}


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- CPU oracle
def oracle_sample_cfg(cfg, target_elems):
    """Same recipe (rank, p, q, noise) on a smaller cube-ish shape of ~target_elems."""
    N = cfg.order
    side = max(int(round(target_elems ** (1.0 / N))), max(cfg.ranks) + cfg.p)
    dims = tuple([side] * N)
    return cfg.scaled(dims, tuple(min(c, side) for c in cfg.core_dims), tuple(min(r, side) for r in cfg.ranks),
                      name=cfg.name + f"-sample{side}")


def run_oracle_steps(cfg, steps, warmup, target_elems):
    import oracle
    scfg = oracle_sample_cfg(cfg, target_elems)
    x = synth.make_tensor(scfg)
    oms = [synth.gaussian_omega(scfg, n) for n in range(scfg.order)]
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        if scfg.algo == "sthosvd":
            om2 = [synth.kron_omegas(scfg, n, synth.sthosvd_dims_before(scfg, n)) for n in range(scfg.order)]
            oracle.sthosvd(x, scfg.ranks, om2, q=scfg.q, kind="kron")
        else:
            oracle.hosvd(x, scfg.ranks, oms, q=scfg.q)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    nbytes = x.size * (8 if scfg.dtype == "f64" else 4)
    return scfg, nbytes, times


def cores_used():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ----------------------------------------------------------------- GPU arm
def run_gpu(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2001_07124_b200 import api as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [P.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    else:
        nid = None
    N = cfg.order
    I_last = cfg.dims[-1]
    if I_last % world:
        raise SystemExit(f"last mode {I_last} not divisible by {world} ranks")
    lo, hi = partition.slab_range(I_last, world, rank)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        X, info = synth.make_tensor_device(cfg, dev, last_range=(lo, hi))
        oms = []
        for n in range(N):
            rows = partition.omega_rows(cfg.dims, n, lo, hi)
            if rows is not None:
                oms.append(synth.gaussian_omega_device(cfg, n, dev, row0=rows[0], rows=rows[1],
                                                       tf32=args.omega == "tf32"))
            else:
                oms.append(synth.gaussian_omega_device(cfg, n, dev, tf32=args.omega == "tf32"))
        torch.cuda.synchronize()
        h = P.Handle(stream=stream, nccl_id=nid, nranks=world, rank=rank)
        if args.omega == "tf32":
            h.set_option(3, 1)              # RT_OPT_OMEGA_TF32: Omega is device-rounded to tf32

        def step():
            return P.rtucker_hosvd(h, X, cfg.ranks, cfg.p, cfg.q, oms, last_offset=lo, last_global=I_last)

        for _ in range(args.warmup):
            res = step()
        h.sync()
        h.profile_read()                    # clear counters
        h.set_option(1, 1)                  # RT_OPT_PROFILE: per-launch CUDA events
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk = ClockSampler(local)
        clk.start()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            res = step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = clk.stop()
        h.set_option(1, 0)
        prof, launches = h.profile_read()
        ms = e0.elapsed_time(e1)
        h.sync()
        E = float(res["err"][0].item())
        Eg = float(res["err"][1].item())
        # ------------------------------------------------ e2e: host buffers through the API
        # Every step copies its inputs (X, Omega) from pinned host memory and reads its result
        # (factors, core, E) back.  Steps are pipelined over two device input buffers: the copy of
        # step k+1 (copy stream) overlaps the decomposition of step k (the transfer-bound stream of
        # decompositions a serving loop runs); the result read of step k follows its compute.
        e2e = None
        if not args.no_e2e:
            xh = torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
            xh.copy_(X)
            omh = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in oms]
            for a, b in zip(omh, oms):
                a.copy_(b)
            X2 = torch.empty_like(X)
            oms2 = [torch.empty_like(o) for o in oms]
            bufs = [(X, oms), (X2, oms2)]
            cstream = torch.cuda.Stream(device=dev)
            ready = [torch.cuda.Event() for _ in range(2)]
            free = [torch.cuda.Event() for _ in range(2)]
            ke = max(2, min(args.steps, args.e2e_steps))
            h2d = xh.numel() * xh.element_size() + sum(o.numel() * o.element_size() for o in omh)
            d2h = 0
            outh = None

            def upload(k):
                xb, ob = bufs[k % 2]
                with torch.cuda.stream(cstream):
                    if k >= 2:
                        cstream.wait_event(free[k % 2])
                    xb.copy_(xh, non_blocking=True)
                    for a, b in zip(ob, omh):
                        a.copy_(b, non_blocking=True)
                    ready[k % 2].record(cstream)

            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            f0 = torch.cuda.Event(enable_timing=True)
            f1 = torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            cstream.wait_stream(stream)
            upload(0)
            for k in range(ke):
                if k + 1 < ke:
                    upload(k + 1)
                xb, ob = bufs[k % 2]
                stream.wait_event(ready[k % 2])
                r2 = P.rtucker_hosvd(h, xb, cfg.ranks, cfg.p, cfg.q, ob, last_offset=lo, last_global=I_last)
                free[k % 2].record(stream)
                res_d = [q for q in r2["Q"]] + [r2["G"], r2["err"]]
                if outh is None:
                    outh = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in res_d]
                for a, b in zip(outh, res_d):
                    a.copy_(b, non_blocking=True)
                d2h = sum(o.numel() * o.element_size() for o in outh)
            f1.record(stream)
            torch.cuda.synchronize()
            e2e_ms = f0.elapsed_time(f1) / ke
            e2e = (e2e_ms, h2d, d2h)
            del X2, oms2
        h.close()
    # ------------------------------------------------------------ reduce over ranks
    t = torch.tensor([ms, e2e[0] if e2e else 0.0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, e2e_ms_max = float(t[0]), float(t[1])
    out = None
    if rank == 0:
        out = dict(ms=ms_max, E=E, Eg=Eg, prof=prof, launches=launches, clocks=clocks,
                   e2e=(e2e_ms_max, e2e[1], e2e[2]) if e2e else None, world=world)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


# the kernels of the residual pass (a8): P chain, residual kernel(s), reductions
RESIDUAL_LABELS = ("residual_tc", "residual_simt", "pchain", "reduce_pairs", "finalize_err", "sumsq", "resid_scale",
                   "split_transpose")


def _pipeline(prof, ms, steps, xbytes):
    """throughput of sketch+QR+core (first sketch to truncated G) with the
    residual pass (a8: P chain + residual kernel) timed and reported separately."""
    res_ms = sum(t for nm, _, t in prof if nm in RESIDUAL_LABELS) / steps
    pm = ms - res_ms
    return {"value": xbytes / (pm * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": pm, "residual_ms": res_ms}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-elems", type=float, default=5.0e8)
    ap.add_argument("--omega", default="tf32", choices=["tf32", "general"],
                    help="tf32: Gaussian Omega rounded to tf32 before the call (RT_OPT_OMEGA_TF32, reading R18, "
                         "2 tensor products per sketch); general: fp32 Gaussian Omega (3 products)")
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # not launched by torchrun: start one rank per GPU ourselves (same command line)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    workload = (f"{cfg.name}: {'x'.join(map(str, cfg.dims))} {cfg.dtype} randomized "
                f"{'HOSVD (Alg.6)' if cfg.algo == 'hosvd' else 'STHOSVD (Alg.8)'}, rank {cfg.ranks}, "
                f"p={cfg.p}, q={cfg.q}, Gaussian Omega, +relative error")
    config = {"workload": workload, "dims": list(cfg.dims), "ranks": list(cfg.ranks), "p": cfg.p, "q": cfg.q,
              "parallelism": f"slab{world}" if world > 1 else "single",
              "omega": ("Gaussian, tf32-rounded on the device before the call (RT_OPT_OMEGA_TF32, reading R18)"
                        if args.omega == "tf32" else "Gaussian fp32 (general Omega: 3xTF32 sketch)"),
              "l2": "inputs larger than L2 (X 32 GiB >> 126 MB; no flush needed)",
              "step": "rtucker_hosvd incl. residual pass for E"}

    if args.impl == "reference":
        if rank != 0:
            return
        target = 6.0e7                  # ~391^3 cube: a few s per step, whole run within minutes
        scfg, nbytes, times = run_oracle_steps(cfg, args.steps, args.warmup, target)
        tot = sum(times)
        val = nbytes * len(times) / tot / 1e9
        line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": dict(config, sample=scfg.name, sample_dims=list(scfg.dims)),
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores_used(), "kind": "oracle",
                                 "sample": f"oracle hosvd on {'x'.join(map(str, scfg.dims))} (same recipe)"},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    r = run_gpu(args, cfg)
    if rank != 0:
        return
    hbm, bf16, bf16s, peak_src = _peaks()
    xbytes = cfg.nbytes
    ms = r["ms"] / args.steps
    value = xbytes / (ms * 1e-3) / 1e9
    wm = work_model(cfg, r["world"], 2 if args.omega == "tf32" else 3)
    # roofline of the X-streaming kernels (the dominant work: every launch that reads X in the
    # sketch+QR+core pipeline; the residual pass a8 is reported apart): algorithmic bytes of those
    # passes (|X| per pass + the test / power matrices and the core stage written)
    # over their device time, CUDA events on the launching stream (RT_OPT_PROFILE)
    prof = sorted(r["prof"], key=lambda e: -e[2])
    # fused passes (one read of X for two contractions): sketch1_core0 = [S1 + G1] (the one-fusion
    # schedule), sketch1_z0 = [Z0 + S1] and sketch2_core0 = [G1 + S2] (the 9-pass schedule)
    fused_labels = ("sketch1_core0", "sketch1_z0", "sketch2_core0")
    xlabels = ("ttm_s_tc", "ttm_s_tc_pow", "ttm_t_tc_pow", "core_first") + fused_labels
    names = {nm for nm, _, _ in prof}
    nfused = sum(1 for f in fused_labels if f in names)
    x_ms = sum(t for nm, _, t in prof if nm in xlabels) / args.steps
    xl = wm["x_bytes_local"]
    npass = wm["ttm_s"][2] + wm["ttm_t"][2] - nfused
    cls_bytes = wm["ttm_s"][0] + wm["ttm_t"][0] - nfused * xl
    cls_flops = wm["ttm_s"][1] + wm["ttm_t"][1]
    roof = None
    if x_ms > 0:
        achieved = cls_bytes / (x_ms * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get("ttm_s_h16")
        roof = {"bound": "hbm", "kernel": "X passes: " + "+".join(xlabels), "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                "traffic_note": "ncu dram bytes read+write per launch of ttm_s_h16_kernel (the most frequent X pass)",
                "algorithmic_bytes_per_pass": cls_bytes / npass, "x_passes_per_step": npass + 1,
                "peak_source": peak_src, "share_of_step": x_ms / ms,
                "tflops": cls_flops / (x_ms * 1e-3) / 1e12}
        # tensor pipe: hardware flops (the first Omega sketch: 2 tf32 products; every other X pass: the
        # 3 fp16-split products, the fused pass 5 per column of its [sketch | core]) against the
        # measured peaks (f16 = measured dense bf16; tf32 = bf16 x 1/2, B200_PROFILING.md's ratio)
        tf32_peak, f16_peak = bf16 / 2.0, bf16
        K0 = cfg.K(0)
        first = 2 * (xl // 4) * K0
        hw_tf32 = 2 * first if args.omega == "tf32" else 3 * first
        hw_f16 = 3 * (cls_flops - first)
        t_s = x_ms * 1e-3
        roof["tensor"] = {"hw_tflops": (hw_tf32 + hw_f16) / t_s / 1e12,
                          "frac": (hw_tf32 / (tf32_peak * 1e12) + hw_f16 / (f16_peak * 1e12)) / t_s,
                          "peak_tflops": {"tf32": tf32_peak, "f16": f16_peak},
                          "peak_source": f"{peak_src} bf16 (f16), x 1/2 (tf32)"}
    line = {"metric": METRIC, "value": value * 1.0, "unit": UNIT, "n_gpus": r["world"], "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
            "ttm_tflops": wm["total_flops"] * r["world"] / (ms * 1e-3) / 1e12,
            "rel_err": r["E"], "rel_err_gram": r["Eg"], "roofline": roof,
            "kernels": [{"name": n, "count": c, "ms_per_step": t / args.steps} for n, c, t in prof[:12]],
            "pipeline": _pipeline(prof, ms, args.steps, xbytes),
            "gpu_launches": int(r["launches"]), "clocks": r["clocks"]}
    if r["e2e"]:
        em, h2d, d2h = r["e2e"]
        line["e2e"] = {"value": xbytes / (em * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(h2d) * r["world"],
                       "d2h_bytes_per_step": int(d2h) * r["world"], "ms_per_step": em}
    if r["world"] == 1 and not args.no_cpu_baseline:
        scfg, nbytes, times = run_oracle_steps(cfg, 1, 0, args.cpu_sample_elems)
        line["cpu_baseline"] = {"value": nbytes / times[0] / 1e9, "unit": UNIT, "cores": cores_used(),
                                "kind": "oracle",
                                "sample": f"fp64 oracle hosvd on {'x'.join(map(str, scfg.dims))} "
                                          f"(same recipe/rank/p/q), {times[0]:.1f} s"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
