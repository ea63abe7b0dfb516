#!/usr/bin/env python
"""Benchmark: unaligned PCG operator applications (matvecs/s) at BASELINE.json config 1.

One "step" = one application of the unaligned normal-equation operator
  y = (F'F + lambda (I kron K) + rho I) x          (unaligned.hpp:101-115)
over all q = 200,000 observations of config 1 (n=200, 100x100 other modes, r=10), i.e. the
PCG hot loop.  `value` is device-timed with inputs resident in HBM and the L2 flushed before
every step (the working set is 3 MB, far below the 126 MB L2); `e2e` is the same metric
through the C-ABI host-buffer call (x uploaded from pinned host memory, y read back each
step).  `roofline` reports the scatter-gather kernel (K1) against the measured HBM peak.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun (N > 1) the observations are sharded over ranks (equal-count slices of the
i_k-sorted set) and the n x r partial accumulator is NCCL all-reduced every step.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK_HBM = 6650.0


def measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return PEAKS_FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def ncu_traffic(kernel_substr):
    """DRAM bytes per launch (read + write) of the named kernel from the committed `ncu --set full`
    capture of this bench's own command (profiles/round*/ncu_full_*.json, newest round first)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "round*", "ncu_full_fused_matvec_config1.json")),
                       reverse=True):
        try:
            caps = [d for d in json.load(open(path)) if kernel_substr in d["kernel"]]
        except Exception:
            continue
        if caps:
            return sum(d["traffic_bytes"] for d in caps) / len(caps), os.path.relpath(path, ROOT)
    return None, None


def alg_bytes_matvec(d, q, n, r):
    """unaligned matvec algorithmic bytes (int32 index stream read once,
    K read twice, six n x r fp64 vectors)."""
    return 4 * d * q + 16 * n * n + 48 * n * r


def alg_bytes_k1(d, q, n, r):
    """Scatter-gather kernel (K1): the d int32 index streams + Xhat rows read + Yhat written."""
    return 4 * d * q + 16 * n * r


def cpu_port_matvec(c, threads, seconds):
    """The oracle's fused streaming restatement on `threads` host cores (test/bench baseline)."""
    import numpy as np
    from oracle import oracle as orc
    from inputs.configs import kernel_matrix
    kern = kernel_matrix(c.points, c.kernel, c.ell)
    factors = [None] + c.factors[1:]
    x = np.random.default_rng(0).normal(size=c.shape[0] * c.r)
    orc.unaligned_matvec_stream(c.shape, 0, c.idx, factors, kern, c.lam, c.rho, x, threads)  # warm
    n_done, t0 = 0, time.perf_counter()
    while True:
        orc.unaligned_matvec_stream(c.shape, 0, c.idx, factors, kern, c.lam, c.rho, x, threads)
        n_done += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return n_done / el, n_done


def secondary(args, ctx, cp, p, c, lib, x, y, stream, flush):
    """Other BASELINE configs and the PCG solve, measured in the same run (N = 1)."""
    import bench_secondary as bs
    sec = {}

    def attempt(key, fn):
        try:
            sec[key] = fn()
        except Exception as e:  # report, never hide: the key carries the failure
            sec[key] = {"error": f"{type(e).__name__}: {e}"}

    attempt("fp64_peak", lambda: bs.fp64_peaks(ctx))
    fp64 = sec["fp64_peak"].get("dmma_tflops", 40.0) if isinstance(sec["fp64_peak"], dict) else 40.0
    attempt("config1_pcg_solve", lambda: bs.config1_pcg(cp, p, c))
    attempt("config1_gram_matvec_ms_l2_flushed", lambda: bs.gram_matvec_ms(p, lib, x, y, stream, flush))
    attempt("config1_precond_apply_ms", lambda: bs.precond_ms(p, lib, c.shape[0], c.r))
    attempt("config0_aligned", lambda: bs.aligned("config0", ctx, 20, fp64))
    attempt("config2_aligned", lambda: bs.aligned("config2", ctx, 10, fp64))
    attempt("als_infinite_update", lambda: bs.als_updates(ctx, p, c))
    if args.large:
        attempt("config3", lambda: bs.large("config3", ctx, fp64_tf=fp64))
        attempt("config4", lambda: bs.large("config4", ctx, fp64_tf=fp64))
    return sec


def run_reference(args, rank):
    if rank != 0:
        return
    from oracle import oracle as orc
    from inputs import configs
    orc.build()
    c = configs.config1()
    threads = orc.max_threads()
    import numpy as np
    from inputs.configs import kernel_matrix
    kern = kernel_matrix(c.points, c.kernel, c.ell)
    factors = [None] + c.factors[1:]
    x = np.random.default_rng(0).normal(size=c.shape[0] * c.r)
    for _ in range(args.warmup):
        orc.unaligned_matvec_stream(c.shape, 0, c.idx, factors, kern, c.lam, c.rho, x, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        orc.unaligned_matvec_stream(c.shape, 0, c.idx, factors, kern, c.lam, c.rho, x, threads)
    el = time.perf_counter() - t0
    v = args.steps / el
    sample = f"config1 full operator application (q=200000) x {args.steps}, fused streaming C port"
    print(json.dumps({
        "impl": "reference", "metric": "unaligned PCG matvecs/s (config 1, q=200k, r=10)", "value": v,
        "unit": "matvecs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config 1)",
        "config": {"workload": "config1: unaligned 200x100x100, q=200000, r=10, lambda=1e-3, rho=1e-6"},
        "cpu_baseline": {"value": v, "unit": "matvecs/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--secondary", type=int, default=1, help="aligned configs 0/2, PCG solves, FP64 peaks")
    ap.add_argument("--large", type=int, default=1, help="configs 3/4 at full size inside --secondary")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2603_25691_b200 as cp
    from paper_2603_25691_b200 import _capi, configs

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _capi.load()
    ctx = cp.Context(local)
    if world > 1:
        uid = [cp.Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_comm(world, rank, uid[0])

    c = configs.config1()
    n, r, d, q = c.shape[0], c.r, len(c.shape), c.idx.shape[1]
    mode = cp.RkhsMode(c.points, c.ell, c.lam, ctx=ctx)
    obs = cp.ObservationSet(c.shape, c.idx, c.vals)
    model = cp.KruskalModel([np.zeros((n, r))] + c.factors[1:])
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, c.rho, shard=rank, shards=world)

    dev = torch.device("cuda", local)
    x = torch.randn(n * r, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)  # 256 MB > 126 MB L2
    ms6 = (ctypes.c_double * 6)()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    def step(ev=None):
        with torch.cuda.stream(stream):
            flush.add_(1)  # evict L2 (outside the events)
            if ev:
                ev[0].record(stream)
            _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
            if ev:
                ev[1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # timed: the K steps captured in ONE CUDA graph (each step = a 256 MB memset node that evicts
    # L2, then the operator between its own event pair) -- how the operator runs inside the
    # device-resident PCG loop.  Plain per-call launches (~4 us host launch cost each on this
    # system, profiles/micro/launch_rate.cu) are measured next to it as value_plain_launch.
    gms = (ctypes.c_float * args.steps)()
    cycle_m = 128
    if world == 1:
        # Timed region: K applications back to back in ONE CUDA graph between one event pair,
        # application t on instance t % 128 of config 1 (its own observation plan, kernel matrix,
        # factors, x, y: ~2 MB touched each, 128 x 2 MB = 2 x the 126 MB L2), so every application starts
        # L2-cold with no flush inside the timed region -- the "inputs larger than L2" option.
        insts = []
        for i in range(cycle_m):
            mi = cp.RkhsMode(c.points, c.ell, c.lam, ctx=ctx)
            oi = cp.ObservationSet(c.shape, c.idx, c.vals)
            pi = cp.make_unaligned_subproblem(oi, model, 0, mi, c.rho)
            xi = torch.randn(n * r, dtype=torch.float64, device=dev)
            insts.append((mi, oi, pi, xi, torch.empty_like(xi)))
        hp = (ctypes.c_void_p * cycle_m)(*[t[2].handle.value for t in insts])
        hx = (ctypes.c_void_p * cycle_m)(*[t[3].data_ptr() for t in insts])
        hy = (ctypes.c_void_p * cycle_m)(*[t[4].data_ptr() for t in insts])
        tot = ctypes.c_float()
        with ClockSampler(local) as clk:
            _capi.check(lib.cphifi_unaligned_matvec_cycle_timed(hp, hx, hy, cycle_m, args.steps, ctypes.byref(tot)))
            torch.cuda.synchronize()
        total_ms = float(tot.value)
        # the per-step flush method (one application between its own events, 256 MB memset node
        # before each, all in one graph) for comparison
        _capi.check(lib.cphifi_unaligned_matvec_graph_timed(p.handle, x.data_ptr(), y.data_ptr(),
                                                            flush.data_ptr(), flush.numel() * 4, args.steps, gms))
        flush_ms = float(sum(gms))
        del insts
    else:  # multi-GPU: NCCL stays outside graph capture; plain launches, per-step L2 flush
        with ClockSampler(local) as clk:
            for i in range(args.steps):
                step(evs[i])
            torch.cuda.synchronize()
        total_ms = flush_ms = float(sum(a.elapsed_time(b) for a, b in evs))
    for i in range(args.steps):
        step(evs[i])
    torch.cuda.synchronize()
    plain_ms = sum(a.elapsed_time(b) for a, b in evs)
    # per-kernel split of the same step (instrumented pass, L2 flushed before each step)
    phases = [0.0] * 6
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.add_(1)
        _capi.check(lib.cphifi_unaligned_matvec_timed(p.handle, x.data_ptr(), y.data_ptr(), 1, ms6))
        phases = [a + b for a, b in zip(phases, ms6)]
    # small n on one GPU the graph step IS the fused kernel (one launch between the events)
    k1_src = total_ms if (world == 1 and n <= 512) else phases[1]
    t = torch.tensor([total_ms, k1_src, plain_ms, flush_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, k1_ms, plain_ms, flush_ms = float(t[0]), float(t[1]), float(t[2]), float(t[3])
    value = args.steps / (total_ms / 1e3)

    # e2e: the reference-facing host-buffer call, H2D of x and D2H of y every step
    hx = torch.randn(n * r, dtype=torch.float64).pin_memory().numpy()
    hy = torch.empty(n * r, dtype=torch.float64).pin_memory().numpy()
    xp, yp = hx.ctypes.data_as(_capi.c_double_p), hy.ctypes.data_as(_capi.c_double_p)
    for _ in range(args.warmup):
        _capi.check(lib.cphifi_unaligned_matvec(p.handle, xp, yp))
    if world > 1:
        dist.barrier()
    e2e_el = 0.0
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.add_(1)
        stream.synchronize()
        t0 = time.perf_counter()
        _capi.check(lib.cphifi_unaligned_matvec(p.handle, xp, yp))
        e2e_el += time.perf_counter() - t0
    te = torch.tensor([e2e_el], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = args.steps / float(te[0])

    # secondary: one full device PCG solve of config 1 (tol 1e-8, max 500)
    rep = cp.SolveReport()
    cp.solve_unaligned_pcg(p, cp.PcgConfig(c.tol, c.max_iter), rep)
    rep2 = cp.SolveReport()
    cp.solve_unaligned_pcg(p, cp.PcgConfig(c.tol, c.max_iter), rep2)

    if rank == 0:
        hbm, src = measured_hbm()
        k1_launch_s = (k1_ms / args.steps) / 1e3
        fused_whole = world == 1 and n <= 512  # one cooperative kernel = the whole operator
        k1_bytes = alg_bytes_matvec(d, q, n, r) if fused_whole else alg_bytes_k1(d, q // world, n, r)
        achieved = k1_bytes / k1_launch_s / 1e9
        traffic, traffic_src = ncu_traffic("fused_matvec_kernel")
        mv_bytes = alg_bytes_matvec(d, q, n, r)
        out = {
            "metric": "unaligned PCG matvecs/s (config 1, q=200k, r=10)",
            "value": value, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "value_flush_per_step": args.steps / (flush_ms / 1e3),
            "value_plain_launch": args.steps / (plain_ms / 1e3),
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config 1)",
            "config": {"workload": "config1: unaligned 200x100x100, q=200000, r=10, lambda=1e-3, rho=1e-6",
                       "l2": ("inputs larger than L2: 128 independent config-1 instances (plan, K, factors, x, y) "
                              "cycled, every application L2-cold; value_flush_per_step = the per-step 256 MB "
                              "flush method" if world == 1 else "flushed before every timed step (256 MB write)"),
                       "timing": ("K applications back to back in one CUDA graph between one CUDA event pair"
                                  if world == 1 else "plain launches, CUDA events around each application"),
                       "parallelism": f"obs-sharded x{world}, n x r all-reduce per step"},
            "roofline": {"bound": "hbm", "kernel": "fused_matvec_kernel (whole operator)" if fused_whole
                         else "fused_matvec_kernel (scatter-gather + fix-up)", "achieved": achieved,
                         "peak": hbm, "peak_source": src, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic, "traffic_source": traffic_src, "alg_bytes_per_launch": k1_bytes,
                         "kernel_ms": k1_ms / args.steps},
            "matvec_hbm_frac": mv_bytes / ((total_ms / args.steps) / 1e3) / 1e9 / hbm,
            "phase_ms": {nm: v / args.steps for nm, v in
                         zip(["K_X_gemm", "fused_kernel", "-", "allreduce", "y_gemm_or_C2", "total"], phases)},
            "e2e": {"value": e2e_value, "unit": "matvecs/s", "h2d_bytes_per_step": 8 * n * r,
                    "d2h_bytes_per_step": 8 * n * r},
            "gpu_launches": (1 if fused_whole else 3) * args.steps,
            "clocks": clk.summary(),
            "pcg_solve": {"iterations": rep2.iterations, "relative_residual": rep2.relative_residual,
                          "wall_s": rep2.wall_time_s, "setup_s": rep2.setup_s, "matvecs": rep2.matvecs},
        }
        if world == 1:
            from oracle import oracle as orc
            threads = orc.max_threads()
            v_cpu, n_cpu = cpu_port_matvec(c, threads, args.cpu_seconds)
            out["cpu_baseline"] = {"value": v_cpu, "unit": "matvecs/s", "cores": threads, "kind": "port",
                                   "sample": f"config1 full operator application (q=200000) x {n_cpu}, "
                                             f"fused streaming C restatement, {threads} threads"}
        if world == 1 and args.secondary:
            out["secondary"] = secondary(args, ctx, cp, p, c, lib, x, y, stream, flush)
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
