#!/usr/bin/env python
"""Benchmark: unaligned PCG operator applications (matvecs/s) at BASELINE.json config 4.

One "step" = one application of the unaligned normal-equation operator
  y = (F'F + lambda (I kron K) + rho I) x          (unaligned.hpp:101-115)
over ALL q = 1e9 draws of config 4 (4096 x 512 x 512, i_1 ~ Zipf(1.1), r = 64): X^ = K X, the
per-observation gather / scatter (observations.hpp:174-198) as one streaming pass over the plan
(the q-pass is inside the timed region: the STREAM operator, not the prebuilt row-Gram form), then
K Y^ + lambda X^ + rho x.  Config 4 is the largest BASELINE config that fits one GPU (BASELINE's
metric names none), so it is the N = 1 workload.

`value` is device-timed (CUDA events on the library stream) with the plan resident in HBM; every
application streams the ~2.9 GB coalesced plan, far above the 126 MB L2 (inputs larger than L2).
`e2e` is the same metric through the reference-facing host-buffer C-ABI call
(cphifi_unaligned_matvec: x copied in from pinned host memory, y read back, every step).
`roofline` is the dominant kernel (the run-structured scatter-gather, k_runs.cu, over the rows
left to it) against the measured HBM peak on SURVEY §8(d)'s per-draw bytes; `roofline_dense_rows`
is the q-pass's second kernel (k_dense_rows.cu: the Zipf-head rows whose cells are mostly drawn,
as FP64 DMMA GEMMs) against the measured DMMA peak; `cpu_baseline` is the oracle's streaming C
port on a bounded sample of the same draws.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun (N > 1) the observations are sharded over ranks (equal-count slices of the i_k-sorted
plan) and the n x r partial accumulator is NCCL all-reduced every application.
"""
from __future__ import annotations

import argparse
import ctypes
import glob
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
METRIC = "unaligned PCG matvecs/s (config 4: q=1e9 draws, 4096x512x512, r=64)"
WORKLOAD = ("config4: unaligned skewed 3-way 4096x512x512, q=1e9 draws (i_1 ~ Zipf(1.1), i_2, i_3 uniform; "
            "coalesced plan of the distinct entries with multiplicities), r=64, lambda=1e-5, rho=1e-6; one step = one "
            "operator application y = (F'F + lambda I(x)K + rho I) x over all q draws (stream operator: the q-pass is "
            "inside the timed region)")
L2_NOTE = ("inputs larger than L2: every application streams the whole config-4 observation set (the GPU arm's "
           "coalesced plan: 2.44e8 entries, ~2.9 GB; the CPU arm's draws) >> the 126 MB L2; no flush")
CONFIG = {"workload": WORKLOAD, "l2": L2_NOTE}  # identical in both arms
DATA = "synthetic (seeded counter-based generator inputs/synth_math.h, BASELINE config 4; the same draws in both arms)"


def measured_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return PEAKS_FALLBACK_HBM, "fallback (B200_PROFILING.md)"


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
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
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


def ncu_traffic(capture, kernel_substr):
    """DRAM bytes per launch (read + write) of the named kernel from the committed `ncu --set full`
    capture of this bench's workload (profiles/round*/<capture>, newest round first)."""
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "round*", capture)), reverse=True):
        try:
            caps = [d for d in json.load(open(path)) if kernel_substr in d["kernel"]]
        except Exception:
            continue
        if caps:
            return sum(d["traffic_bytes"] for d in caps) / len(caps), os.path.relpath(path, ROOT)
    return None, None


def alg_bytes_matvec(d, q, n, r):
    """unaligned matvec algorithmic bytes on the as-given draws (int32 index stream read
    once, K read twice, six n x r fp64 vectors)."""
    return 4 * d * q + 16 * n * n + 48 * n * r


def alg_flops_matvec(d, q, n, r):
    return (d + 2) * r * q + 4 * n * n * r


def alg_bytes_k1(d, q, n, r):
    """Streaming scatter-gather kernel: the d int32 index streams + Xhat rows read + Yhat written."""
    return 4 * d * q + 16 * n * r


# ---- CPU side (the oracle's streaming port; test infrastructure, never the measured GPU path) ------
def cpu_config4_sample(threads, q_sample, reps_target_s, seed_off=0):
    """Time the oracle's fused streaming restatement (oracle/cphifi_oracle.c, SURVEY §8c mode ii) on
    config 4: the dense part (K X, K Yhat, axpys) timed whole, the per-observation pass on draws
    [off, off + q_sample) of the same generator, extrapolated to q = 1e9 draws.
    Returns (seconds per application, detail dict)."""
    import numpy as np

    from inputs import configs
    from oracle import oracle as orc
    cfg = configs.config4()
    n, r = cfg.shape[0], cfg.r
    idx, _ = configs.generate_host(cfg, seed_off, seed_off + q_sample, values=False, threads=threads)
    kern = orc.gaussian_kernel(cfg.points, cfg.ell)
    factors = [None] + cfg.factors[1:]
    x = np.random.default_rng(0).normal(size=n * r)
    empty = np.zeros((3, 0), dtype=np.int32)
    t0 = time.perf_counter()
    orc.unaligned_matvec_stream(cfg.shape, 0, empty, factors, kern, cfg.lam, cfg.rho, x, threads)
    t_dense = time.perf_counter() - t0
    xhat = np.asfortranarray(np.random.default_rng(1).normal(size=(n, r)))
    orc.scatter_gather_stream(cfg.shape, 0, idx[:, : min(q_sample, 200_000)], factors, xhat, threads)  # warm
    reps, t0 = 0, time.perf_counter()
    while True:
        orc.scatter_gather_stream(cfg.shape, 0, idx, factors, xhat, threads)
        reps += 1
        if time.perf_counter() - t0 >= reps_target_s:
            break
    t_stream = (time.perf_counter() - t0) / reps
    per_app = t_dense + t_stream * (cfg.q / q_sample)
    return per_app, {"t_dense_s": t_dense, "t_stream_sample_s": t_stream, "q_sample": q_sample, "reps": reps}


def run_reference(args, rank):
    """The reference arm: the reference CPU path restated (the reference itself, header-only C++ over
    Eigen, cannot be built here: SURVEY §8c), i.e. the oracle's streaming port, on all host cores, on
    config 4 — inputs from inputs/ (never the product library)."""
    if rank != 0:
        return
    from oracle import oracle as orc
    orc.build()
    threads = orc.max_threads()
    q_sample = args.cpu_sample
    for w in range(args.warmup):
        cpu_config4_sample(threads, min(q_sample, 2_000_000), 0.0, seed_off=w * q_sample)
    dense, stream = [], []
    for s in range(args.steps):
        _, det = cpu_config4_sample(threads, q_sample, 0.0, seed_off=s * q_sample)
        dense.append(det["t_dense_s"])
        stream.append(det["t_stream_sample_s"])
    t_app = statistics.mean(dense) + statistics.mean(stream) * (1e9 / q_sample)
    v = 1.0 / t_app
    sample = (f"config 4, each step: the dense part (2 x 4096^2 x 64 GEMMs + axpys) timed whole plus the per-"
              f"observation streaming pass on {q_sample} consecutive draws of the 1e9 (step s: draws [s*{q_sample}, "
              f"(s+1)*{q_sample})), extrapolated x{1e9 / q_sample:.0f}; oracle/cphifi_oracle.c fused streaming "
              f"restatement, {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "matvecs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_app, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": CONFIG, "parallelism": f"CPU, {threads} threads",
        "timing": "wall clock (perf_counter) around each sampled step",
        "cpu_baseline": {"value": v, "unit": "matvecs/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "matvecs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": {"t_dense_s_mean": statistics.mean(dense), "t_stream_sample_s_mean": statistics.mean(stream)},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline: seconds of streaming work")
    ap.add_argument("--cpu-sample", type=int, default=20_000_000, help="CPU baseline: draws per sample")
    ap.add_argument("--secondary", type=int, default=1, help="PCG solves, configs 0-3, CPU baselines 0-3")
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
    from inputs import configs
    from paper_2603_25691_b200 import _capi

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _capi.load()
    ctx = cp.Context(local)
    if world > 1:
        uid = [cp.Context.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.init_comm(world, rank, uid[0])
    dev = torch.device("cuda", local)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)

    cfg = configs.config4()
    n, r, d, q = cfg.shape[0], cfg.r, len(cfg.shape), cfg.q
    t0 = time.perf_counter()
    idx, vals = cp.synth_observations_device(cfg, ctx)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), q, keepalive=(idx, vals),
                                coalesce=cfg.coalesce)
    model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
    t0 = time.perf_counter()
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho, shard=rank, shards=world)
    plan_s = time.perf_counter() - t0
    qt, ql = ctypes.c_int64(), ctypes.c_int64()
    _capi.check(lib.cphifi_obs_info(obs.plan(0, ctx, rank, world).h, ctypes.byref(qt), ctypes.byref(ql), None))
    del idx, vals
    obs.release_inputs()
    torch.cuda.empty_cache()
    p.set_operator("stream")  # the q-pass inside every application

    x = torch.randn(n * r, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)

    def app():
        _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))

    for _ in range(args.warmup):
        app()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                app()
            e1.record(stream)
        torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()

    # the dominant kernel: per-phase device times of the same application (events around each phase)
    ms6 = (ctypes.c_double * 6)()
    _capi.check(lib.cphifi_unaligned_matvec_timed(p.handle, x.data_ptr(), y.data_ptr(), min(args.steps, 10), ms6))
    launches = ctypes.c_int()
    _capi.check(lib.cphifi_unaligned_matvec_launches(p.handle, x.data_ptr(), y.data_ptr(), ctypes.byref(launches)))
    qplan = p.qpass_plan()
    dfma, dmma = ctypes.c_double(), ctypes.c_double()
    _capi.check(lib.cphifi_fp64_peak(ctx.handle, ctypes.byref(dfma), ctypes.byref(dmma)))

    # e2e: the reference-facing host-buffer call, x in from pinned host memory and y back, every step
    hx = torch.randn(n * r, dtype=torch.float64).pin_memory().numpy()
    hy = torch.empty(n * r, dtype=torch.float64).pin_memory().numpy()
    xp, yp = hx.ctypes.data_as(_capi.c_double_p), hy.ctypes.data_as(_capi.c_double_p)
    for _ in range(args.warmup):
        _capi.check(lib.cphifi_unaligned_matvec(p.handle, xp, yp))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _capi.check(lib.cphifi_unaligned_matvec(p.handle, xp, yp))
    e2e_s = time.perf_counter() - t0

    t = torch.tensor([total_ms, ms6[1], ms6[5], e2e_s, ms6[2]], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, k1_ms, app_ms_phased, e2e_s, dense_ms = (float(v) for v in t)
    value = args.steps / (total_ms / 1e3)
    # per-rank q-pass shares (cost-balanced shards give the head ranks the dense rows and the tail ranks the
    # sparse rows): the rooflines below describe the rank whose kernel took longest
    mine = torch.tensor([ms6[1], ms6[2], qplan["sparse_draws"], qplan["parts"], qplan["dense_rows"],
                         qplan["sparse_entries_unpadded"], ql.value, ms6[5]], dtype=torch.float64, device=dev)
    per_rank = [mine]
    if world > 1:
        per_rank = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(per_rank, mine)
    per_rank = [[float(v) for v in pr.tolist()] for pr in per_rank]
    jr = max(range(len(per_rank)), key=lambda j: per_rank[j][0])  # the rank with the slowest run kernel
    jd = max(range(len(per_rank)), key=lambda j: per_rank[j][1])  # ... the slowest dense-rows kernel
    qplan = dict(qplan, sparse_draws=int(per_rank[jr][2]), parts=int(per_rank[jr][3]),
                 sparse_entries_unpadded=int(per_rank[jr][5]), dense_rows=int(per_rank[jd][4]))
    k1_ms, dense_ms = per_rank[jr][0], per_rank[jd][1]

    sec = {}
    if rank == 0 and world == 1 and args.secondary:
        import bench_secondary as bs
        sec = bs.run_all(args, ctx, cp, p, mode, cfg, t1_ms=total_ms / args.steps)
    del p
    torch.cuda.empty_cache()

    if rank == 0:
        hbm, hbm_src = measured_hbm()
        fp64 = sec.get("fp64_peak", {}).get("dmma_tflops") if isinstance(sec.get("fp64_peak"), dict) else None
        # the q-pass = the run kernel over the plan's parts (one launch per factor-block part) + the
        # dense-rows kernel (k_dense_rows.cu, rows whose cells are mostly drawn, as DMMA GEMMs)
        nparts = max(1, qplan["parts"])
        sparse_draws = qplan["sparse_draws"] if qplan["sparse_draws"] >= 0 else q // world
        k1_bytes = alg_bytes_k1(d, sparse_draws, n, r) / nparts  # per launch
        k1_launch_s = k1_ms / 1e3 / nparts
        achieved = k1_bytes / k1_launch_s / 1e9
        traffic, traffic_src = ncu_traffic("ncu_full_runs_config4.json", "runs_kernel")
        nd = qplan["dense_rows"]
        n1, n2 = cfg.shape[1], cfg.shape[2]
        dense_flops = 4.0 * nd * n1 * n2 * r  # two GEMMs per dense row: S = U A_2', P = T A_2 (2 flops / FMA)
        dtraffic, dtraffic_src = ncu_traffic("ncu_full_dense_config4.json", "dense_rows_kernel")
        t_app = total_ms / args.steps / 1e3
        clk_sum = clk.summary()
        clk_mhz = clk_sum.get("sm_mhz") or clk_sum.get("sm_max_mhz") or 1965.0
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        smem_peak = 128.0 * sms * clk_mhz * 1e6 / 1e9
        smem_bytes = qplan["sparse_entries_unpadded"] * (d - 2) * 8.0 * r / nparts
        b_alg, f_alg = alg_bytes_matvec(d, q, n, r), alg_flops_matvec(d, q, n, r)
        qpass_bytes = alg_bytes_k1(d, q // world, n, r)
        out = {
            "metric": METRIC, "value": value, "unit": "matvecs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": CONFIG,
            "timing": "K applications back to back on the library stream between one CUDA event pair",
            "parallelism": (f"observations sharded x{world} (cost-balanced row-aligned slices of the sorted plan), "
                            "each rank contracts its own rows of K, one n x r all-reduce per application")
            if world > 1 else "1 GPU",
            "plan_entries_this_rank": ql.value,
            "qpass_plan": qplan,
            "per_rank": [{"rank": j, "runs_kernel_ms": pr[0], "dense_rows_kernel_ms": pr[1], "sparse_draws": int(pr[2]),
                          "dense_rows": int(pr[4]), "plan_entries": int(pr[6]), "application_ms": pr[7]}
                         for j, pr in enumerate(per_rank)],
            "roofline": {"bound": "hbm", "kernel": f"runs_kernel (k_runs.cu: the per-entry gather / scatter over the "
                                                  f"sparse rows, {nparts} launches per application, one per "
                                                  f"factor-block part)",
                         "achieved": achieved, "peak": hbm, "peak_source": hbm_src, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                         "alg_bytes_per_launch": k1_bytes,
                         "alg_bytes_note": "SURVEY 8(d) per-draw bytes (4 d: the int32 index stream) x the draws of "
                                           "the run kernel's rows (qpass_plan.sparse_draws), + 16 n r (Xhat read, "
                                           "Yhat written), per launch; traffic = ncu DRAM bytes per launch (the "
                                           "coalesced plan streams 12 B per distinct entry)",
                         "kernel_ms_per_launch": k1_launch_s * 1e3, "kernel_ms_per_application": k1_ms,
                         "kernel_share_of_step": k1_ms / app_ms_phased},
            # the run kernel is bound by the shared-memory crossbar, not HBM: every entry reads its staged
            # factor rows (the first other mode is hoisted per run) — (d - 2) x 8 r bytes per entry —
            # against 128 B/clk/SM (B300_MICROARCH.md "smem crossbar BW") x SMs x the sampled SM clock
            "roofline_smem": {"bound": "smem", "kernel": "runs kernel (per-entry factor-row reads)",
                              "achieved": smem_bytes / k1_launch_s / 1e9, "peak": smem_peak, "unit": "GB/s",
                              "frac": smem_bytes / k1_launch_s / 1e9 / smem_peak,
                              "alg_bytes_per_launch": smem_bytes,
                              "peak_note": f"128 B/clk/SM x {sms} SMs x {clk_mhz:.0f} MHz (sampled median SM clock)"},
            "roofline_dense_rows": {"bound": "tensor", "kernel": "dense_rows_kernel (k_dense_rows.cu: the rows whose "
                                                                 "cells are mostly drawn, two FP64 DMMA GEMMs per row)",
                                    "achieved": dense_flops / (dense_ms / 1e3) / 1e12 if dense_ms > 0 else None,
                                    "peak": dmma.value, "peak_source": "measured FP64 DMMA (cphifi_fp64_peak, this run)",
                                    "unit": "TFLOP/s",
                                    "frac": (dense_flops / (dense_ms / 1e3) / 1e12 / dmma.value) if dense_ms > 0 else None,
                                    "traffic": dtraffic, "traffic_source": dtraffic_src,
                                    "alg_flops_per_launch": dense_flops, "dense_rows": nd,
                                    "kernel_ms": dense_ms, "kernel_share_of_step": dense_ms / app_ms_phased},
            "qpass_as_given": {"alg_bytes": qpass_bytes, "ms": k1_ms + dense_ms,
                               "hbm_frac": qpass_bytes / ((k1_ms + dense_ms) / 1e3) / 1e9 / hbm,
                               "note": "the whole q-pass (both kernels) on SURVEY 8(d)'s as-given bytes 4 d q + 16 n r"},
            "fp64": {"alg_flops_per_application": f_alg,
                     "achieved_tflops": f_alg / t_app / 1e12, "peak_tflops_dmma_measured": fp64,
                     "survey_roofline_frac": (max(b_alg / (hbm * 1e9), f_alg / (fp64 * 1e12)) / t_app) if fp64 else None,
                     "note": "SURVEY 8(d): t_roof = max(B_alg/HBM, F_alg/P_FP64) on the as-given q draws; dedup of "
                             "repeated draws and the hoisted first mode make the executed flops lower"},
            "matvec_hbm_frac": b_alg / t_app / 1e9 / hbm,
            "phase_ms": {nm: ms6[i] for i, nm in enumerate(["K_X_gemm", "runs_kernel", "dense_rows_kernel",
                                                            "allreduce", "y_gemm", "whole_application"])},
            "e2e": {"value": args.steps / e2e_s, "unit": "matvecs/s", "h2d_bytes_per_step": 8 * n * r,
                    "d2h_bytes_per_step": 8 * n * r,
                    "call": "cphifi_unaligned_matvec (host x in, host y out, synchronous)"},
            "gpu_launches": launches.value * args.steps,
            "gpu_launches_per_step": launches.value,
            "clocks": clk_sum,
            "setup": {"generate_s": gen_s, "plan_s": plan_s, "q_total": qt.value, "plan_entries_this_rank": ql.value},
        }
        if world == 1:
            from oracle import oracle as orc
            threads = orc.max_threads()
            t_cpu, det = cpu_config4_sample(threads, args.cpu_sample, args.cpu_seconds)
            out["cpu_baseline"] = {
                "value": 1.0 / t_cpu, "unit": "matvecs/s", "cores": threads, "kind": "port",
                "sample": f"config 4: dense part timed whole + streaming pass over {args.cpu_sample} of the 1e9 draws "
                          f"(x{det['reps']} for {args.cpu_seconds:.0f} s), extrapolated to q = 1e9; oracle/cphifi_"
                          f"oracle.c fused streaming restatement, {threads} threads", "detail": det}
        if sec:
            out["secondary"] = sec
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
