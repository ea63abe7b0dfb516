"""Secondary measurements reported inside bench.py's JSON line (N = 1 only): the config-4 PCG solves
(stream and row-Gram operators, the G build counted in the solve), configs 0-3 on device, the ALS
updates, and CPU baselines for configs 0-3 (the oracle's ports, core counts stated).

Everything is device-timed with CUDA events on the library stream unless stated; numbers that
use the row-Gram operator are labelled as such (it reads G, not the observations, per
application, so its roofline is computed on its own bytes, not the as-given per-observation
bytes of SURVEY §8d).
"""
from __future__ import annotations

import ctypes
import json
import os
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def fp64_peaks(ctx):
    from paper_2603_25691_b200 import _capi
    a, b = ctypes.c_double(), ctypes.c_double()
    _capi.call("cphifi_fp64_peak", ctx.handle, ctypes.byref(a), ctypes.byref(b))
    return {"dfma_tflops": a.value, "dmma_tflops": b.value}


def aligned(which, ctx, iters, fp64_tf):
    """Aligned solve (MTTKRP + Gram + decoupled rotate/divide/rotate; eig(V) reported as setup)."""
    import paper_2603_25691_b200 as cp
    from paper_2603_25691_b200 import _capi
    from inputs import configs
    c = getattr(configs, which)()
    n, r = c.shape[0], c.r
    mode = cp.RkhsMode(c.points, c.ell, c.lam, ctx=ctx)
    t0 = time.perf_counter()
    mode.eig()
    eig_k_s = time.perf_counter() - t0
    t = cp.DenseTensor(c.shape, c.tensor)
    dt = cp._device_tensor(t, ctx)
    model = cp.KruskalModel([np.zeros((n, r))] + c.factors[1:])
    arrs, ptrs = cp._factor_array(model.factors, 0)
    w = np.zeros((n, r), order="F")
    ms = (ctypes.c_double * 5)()
    _capi.call("cphifi_aligned_solve_timed", dt.handle, mode.handle, 0, r, ptrs, iters, w.ctypes.data_as(_capi.c_double_p),
               ms)
    N = int(np.prod(c.shape))
    b_alg = 8 * N + 16 * n * n + 32 * n * r
    f_alg = 2 * N * r + 4 * n * n * r + 4 * n * r * r
    t_s = ms[4] / 1e3
    hbm = hbm_peak()
    t_roof = max(b_alg / (hbm * 1e9), f_alg / (fp64_tf * 1e12))
    return {"solves_per_s": 1.0 / t_s, "solve_ms": ms[4], "mttkrp_ms": ms[0], "gram_ms": ms[1],
            "eigV_setup_ms": ms[2], "decoupled_ms": ms[3], "eigK_setup_s": eig_k_s,
            "alg_bytes": b_alg, "alg_flops": f_alg, "hbm_frac": b_alg / t_s / 1e9 / hbm,
            "fp64_tflops": f_alg / t_s / 1e12, "roofline_frac": t_roof / t_s,
            "note": "tensor device-resident; L2 " + ("flushed implicitly (537 MB tensor > L2)" if N * 8 > 2**27
                                                     else "warm (16 MB tensor < L2)")}


def large(which, ctx, iters=3, solve=True, fp64_tf=None):
    """Configs 3/4 at full size: per-observation operator, row-Gram operator, PCG (row-Gram).
    Config 4's plan coalesces repeated draws (cfg.coalesce): the streamed entries are the distinct
    multi-indices, the algorithmic bytes / flops below stay those of the as-given q draws."""
    import torch

    import paper_2603_25691_b200 as cp
    from paper_2603_25691_b200 import _capi
    from inputs import configs
    cfg = getattr(configs, which)()
    n, r, d, q = cfg.shape[0], cfg.r, len(cfg.shape), cfg.q
    lib = _capi.load()
    t0 = time.perf_counter()
    idx, vals = cp.synth_observations_device(cfg, ctx)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), q, keepalive=(idx, vals),
                                coalesce=cfg.coalesce)
    model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
    t0 = time.perf_counter()
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho)
    plan_s = time.perf_counter() - t0
    p.set_operator("stream")
    qt, ql = ctypes.c_int64(), ctypes.c_int64()
    _capi.check(lib.cphifi_obs_info(obs.plan(0, ctx).h, ctypes.byref(qt), ctypes.byref(ql), None))
    del idx, vals
    obs.release_inputs()
    torch.cuda.empty_cache()
    dev = torch.device("cuda", ctx.device)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    x = torch.randn(n * r, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)

    def timed(k):
        ts = []
        for _ in range(k):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                a.record(stream)
                _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
                b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    timed(1)
    stream_ms = timed(iters)
    t0 = time.perf_counter()
    p.set_operator("gram")
    timed(1)
    gram_build_s = time.perf_counter() - t0
    gram_ms = timed(max(5, iters))
    hbm = hbm_peak()
    b_alg = 4 * d * q + 16 * n * n + 48 * n * r
    rp = max(4, 1 << (r - 1).bit_length())
    b_gram = 16 * n * n + 8 * n * rp * rp + 48 * n * r
    f_alg = (d + 2) * r * q + 4 * n * n * r
    if fp64_tf is None:
        fp64_tf = fp64_peaks(ctx)["dmma_tflops"]
    t_roof = max(b_alg / (hbm * 1e9), f_alg / (fp64_tf * 1e12))
    out = {"q": q, "gen_s": gen_s, "plan_s": plan_s, "coalesced": cfg.coalesce, "plan_entries": ql.value,
           "stream_matvec_ms": stream_ms, "stream_matvecs_per_s": 1e3 / stream_ms,
           "stream_hbm_frac_as_given": b_alg / (stream_ms / 1e3) / 1e9 / hbm,
           "stream_roofline_frac_survey": t_roof / (stream_ms / 1e3),
           "roofline_note": "SURVEY 8(d): t_roof = max(B_alg/HBM, F_alg/P_FP64(DMMA, measured)), as-given q",
           "gram_build_s": gram_build_s, "gram_matvec_ms": gram_ms, "gram_matvecs_per_s": 1e3 / gram_ms,
           "gram_hbm_frac_own_bytes": b_gram / (gram_ms / 1e3) / 1e9 / hbm}
    if solve:
        t0 = time.perf_counter()
        mode.eig()
        out["eigK_s"] = time.perf_counter() - t0
        out["precond_apply_ms"] = precond_ms(p, lib, n, r)
        rep = cp.SolveReport()
        cp.solve_unaligned_pcg(p, cp.PcgConfig(cfg.tol, cfg.max_iter), rep)
        out["pcg_gram"] = {"iterations": rep.iterations, "relative_residual": rep.relative_residual,
                           "converged": rep.converged, "wall_s": rep.wall_time_s,
                           "note": "first solve: includes the device-loop graph capture"}
        rep = cp.SolveReport()
        cp.solve_unaligned_pcg(p, cp.PcgConfig(cfg.tol, cfg.max_iter), rep)
        out["pcg_gram_repeat"] = {"iterations": rep.iterations, "relative_residual": rep.relative_residual,
                                  "converged": rep.converged, "wall_s": rep.wall_time_s}
    del p, obs
    torch.cuda.empty_cache()
    return out


def precond_ms(p, lib, n, r, iters=20):
    """Device time of one preconditioner application M^-1 x (unaligned.hpp:135-139), reported
    per PCG iteration next to the operator."""
    import torch
    from paper_2603_25691_b200 import _capi
    import paper_2603_25691_b200 as cp
    dev = torch.device("cuda", 0)
    x = torch.randn(n * r, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    cp.build_preconditioner(p)  # eig(V), D (setup)
    _capi.check(lib.cphifi_unaligned_precond_apply_device(p.handle, x.data_ptr(), y.data_ptr()))
    stream = torch.cuda.ExternalStream(p.mode.ctx.stream(), device=dev)
    ts = []
    for _ in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            _capi.check(lib.cphifi_unaligned_precond_apply_device(p.handle, x.data_ptr(), y.data_ptr()))
            b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def config4_solves(cp, p, obs, mode, cfg):
    """Config 4 PCG solves on the headline plan: the stream operator (the reference's structure), the
    row-Gram operator (drop-in default; G built inside the solve's setup), and a fresh-factor solve
    (a new subproblem on the same observation plan: B, V, G, eig(V), PCG — one ALS infinite-mode
    update's worth of work, unaligned.hpp:35-48 + 143-161)."""
    import numpy as np
    out = {}
    pc = cp.PcgConfig(cfg.tol, cfg.max_iter)
    for op in ("stream", "gram"):
        p.set_operator(op)
        rep = cp.SolveReport()
        t0 = time.perf_counter()
        cp.solve_unaligned_pcg(p, pc, rep)
        first = time.perf_counter() - t0
        rep2 = cp.SolveReport()
        cp.solve_unaligned_pcg(p, pc, rep2)
        out[op] = {"iterations": rep.iterations, "relative_residual": rep.relative_residual,
                   "first_wall_s": first, "first_setup_s": rep.setup_s, "repeat_wall_s": rep2.wall_time_s,
                   "repeat_iterations": rep2.iterations}
    n, r = cfg.shape[0], cfg.r
    g = np.random.default_rng(5)
    fac = [np.zeros((n, r))] + [f * (1.0 + 0.01 * g.normal(size=f.shape)) for f in cfg.factors[1:]]
    t0 = time.perf_counter()
    p2 = cp.make_unaligned_subproblem(obs, cp.KruskalModel(fac), 0, mode, cfg.rho)
    t_sub = time.perf_counter() - t0
    rep = cp.SolveReport()
    cp.solve_unaligned_pcg(p2, pc, rep)
    out["fresh_factors_gram"] = {"subproblem_s": t_sub, "pcg_wall_s": rep.wall_time_s, "pcg_setup_s": rep.setup_s,
                                 "iterations": rep.iterations, "relative_residual": rep.relative_residual,
                                 "total_s": t_sub + rep.wall_time_s, "operator": p2.operator(),
                                 "note": "plan reused, fresh other-mode factors: B (one stream pass with the "
                                         "values), V, G build, eig(V), preconditioner, PCG"}
    p.set_operator("stream")
    return out


def config4_shards(cp, ctx, mode, cfg, t1_ms, counts=(2, 4, 8), iters=10):
    """Config 4 cut into S cost-balanced observation shards (capi.cu balanced_shard_cuts), each
    shard's row-sharded operator application timed ALONE on this GPU (one shard at a time, no
    communicator: the call returns the shard's partial y_s).  The slowest shard bounds the S-GPU
    application; the n x r all-reduce of the partials (2 MB over NVLink) is NOT in these times."""
    import numpy as np
    import torch
    from paper_2603_25691_b200 import _capi
    lib = _capi.load()
    dev = torch.device("cuda", ctx.device)
    n, r, q = cfg.shape[0], cfg.r, cfg.q
    idx, vals = cp.synth_observations_device(cfg, ctx)
    model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
    x = torch.randn(n * r, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    out = {"t1_ms": t1_ms, "note": "every shard timed alone on one GPU; all-reduce of the n x r partials not included"}
    for S in counts:
        ms = []
        for s in range(S):
            obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), q, keepalive=(idx, vals),
                                        coalesce=cfg.coalesce)
            p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho, shard=s, shards=S)
            p.set_operator("stream")
            for _ in range(3):
                _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(iters):
                    _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
                e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1) / iters)
            del p, obs
            torch.cuda.empty_cache()
        out[f"S{S}"] = {"shard_ms": ms, "max_ms": max(ms), "projected_speedup": t1_ms / max(ms)}
    del idx, vals
    torch.cuda.empty_cache()
    return out


def config1_line(cp, ctx, steps):
    """Config 1 operator (the previous round's headline) on 128 independent instances cycled in one
    CUDA graph (>= 128 applications so every application starts L2-cold), and its PCG solve."""
    import numpy as np
    import torch
    from inputs import configs
    from paper_2603_25691_b200 import _capi
    lib = _capi.load()
    c = configs.config1()
    n, r = c.shape[0], c.r
    dev = torch.device("cuda", ctx.device)
    model = cp.KruskalModel([np.zeros((n, r))] + c.factors[1:])
    m = 128
    insts = []
    for _ in range(m):
        mi = cp.RkhsMode(c.points, c.ell, c.lam, ctx=ctx)
        oi = cp.ObservationSet(c.shape, c.idx, c.vals)
        pi = cp.make_unaligned_subproblem(oi, model, 0, mi, c.rho)
        xi = torch.randn(n * r, dtype=torch.float64, device=dev)
        insts.append((mi, oi, pi, xi, torch.empty_like(xi)))
    k = max(steps, 2 * m)
    hp = (ctypes.c_void_p * m)(*[t[2].handle.value for t in insts])
    hx = (ctypes.c_void_p * m)(*[t[3].data_ptr() for t in insts])
    hy = (ctypes.c_void_p * m)(*[t[4].data_ptr() for t in insts])
    tot = ctypes.c_float()
    _capi.check(lib.cphifi_unaligned_matvec_cycle_timed(hp, hx, hy, m, k, ctypes.byref(tot)))
    p = insts[0][2]
    xh = np.random.default_rng(0).normal(size=n * r)
    for _ in range(5):
        cp.unaligned_matvec(p, xh)
    t0 = time.perf_counter()
    for _ in range(200):
        cp.unaligned_matvec(p, xh)
    e2e = 200 / (time.perf_counter() - t0)
    rep = cp.SolveReport()
    cp.solve_unaligned_pcg(p, cp.PcgConfig(c.tol, c.max_iter), rep)
    rep = cp.SolveReport()
    cp.solve_unaligned_pcg(p, cp.PcgConfig(c.tol, c.max_iter), rep)
    return {"matvecs_per_s": k / (tot.value / 1e3), "applications": k, "e2e_matvecs_per_s": e2e,
            "pcg": {"iterations": rep.iterations, "relative_residual": rep.relative_residual,
                    "wall_s": rep.wall_time_s},
            "note": "128 independent config-1 instances cycled in one CUDA graph (>= 2 cycles: every application "
                    "L2-cold); e2e = cphifi_unaligned_matvec with host buffers"}


def cpu_baselines(threads):
    """The oracle's CPU restatements: reference-faithful on 1 core (configs 0-2:
    materialised Zhat / unfold + Khatri-Rao, two passes) and the fused streaming port on all host
    cores (configs 1, 3; config 4 is the headline's cpu_baseline).  Same seeded inputs, same units."""
    import numpy as np
    from inputs import configs
    from oracle import oracle as orc
    out = {}

    def timed(fn, min_s=2.0, max_reps=50):
        fn()
        reps, t0 = 0, time.perf_counter()
        while reps < max_reps:
            fn()
            reps += 1
            if time.perf_counter() - t0 >= min_s:
                break
        return (time.perf_counter() - t0) / reps

    for which in ("config0", "config2"):
        c = getattr(configs, which)()
        n, r = c.shape[0], c.r
        kern = orc.gaussian_kernel(c.points, c.ell)
        ek = orc.sym_eig(kern)
        fac = [np.zeros((n, r))] + c.factors[1:]
        t3 = c.tensor.reshape(c.shape, order="F")

        def solve():
            b = orc.mttkrp(t3, fac, 0, threads=1)
            v = orc.gram_khatri_rao(fac, 0)
            return orc.solve_aligned_decoupled(b, ek, orc.sym_eig(v), c.lam, threads=1)
        t = timed(solve, min_s=2.0, max_reps=5 if which == "config2" else 50)
        out[which] = {"solves_per_s": 1.0 / t, "cores": 1, "kind": "port (reference-faithful: unfold copy, "
                      "materialised Khatri-Rao, GEMM, decoupled solve; eig(K) setup excluded)"}
    c = configs.config1()
    n, r = c.shape[0], c.r
    kern = orc.gaussian_kernel(c.points, c.ell)
    fac = [np.zeros((n, r))] + c.factors[1:]
    sub = orc.make_unaligned_subproblem(c.shape, c.idx, c.vals, fac, 0, kern, c.lam, c.rho)
    x = np.random.default_rng(0).normal(size=n * r)
    t_ref = timed(lambda: orc.unaligned_matvec(sub, x, 1))
    t_str = timed(lambda: orc.unaligned_matvec_stream(c.shape, 0, c.idx, fac, kern, c.lam, c.rho, x, threads))
    out["config1"] = {"ref_1core_matvecs_per_s": 1.0 / t_ref, "stream_matvecs_per_s": 1.0 / t_str,
                      "stream_cores": threads}
    c3 = configs.config3()
    qs = 10_000_000
    idx, _ = configs.generate_host(c3, 0, qs, values=False, threads=threads)
    kern3 = orc.matern32_kernel(c3.points, c3.ell)
    fac3 = [None] + c3.factors[1:]
    x3 = np.random.default_rng(0).normal(size=c3.shape[0] * c3.r)
    empty = np.zeros((4, 0), dtype=np.int32)
    t_dense = timed(lambda: orc.unaligned_matvec_stream(c3.shape, 0, empty, fac3, kern3, c3.lam, c3.rho, x3, threads),
                    min_s=0.5, max_reps=3)
    xh = np.asfortranarray(np.random.default_rng(1).normal(size=(c3.shape[0], c3.r)))
    t_s = timed(lambda: orc.scatter_gather_stream(c3.shape, 0, idx, fac3, xh, threads), min_s=3.0, max_reps=10)
    out["config3"] = {"stream_matvecs_per_s": 1.0 / (t_dense + t_s * c3.q / qs), "stream_cores": threads,
                      "sample": f"dense part timed whole + streaming pass over {qs} of the 2e8 draws, extrapolated"}
    return out


def run_all(args, ctx, cp, p, mode, cfg, t1_ms=None):
    """Everything above, each failure reported in its key (never hidden)."""
    import torch
    from oracle import oracle as orc
    sec = {}

    def attempt(key, fn):
        try:
            sec[key] = fn()
        except Exception as e:  # report, never hide: the key carries the failure
            sec[key] = {"error": f"{type(e).__name__}: {e}"}

    attempt("fp64_peak", lambda: fp64_peaks(ctx))
    fp64 = sec["fp64_peak"].get("dmma_tflops", 40.0) if isinstance(sec["fp64_peak"], dict) else 40.0
    obs = p.obs
    attempt("config4_pcg", lambda: config4_solves(cp, p, obs, mode, cfg))
    torch.cuda.empty_cache()
    if t1_ms:
        attempt("config4_shards", lambda: config4_shards(cp, ctx, mode, cfg, t1_ms))
    attempt("config3", lambda: large("config3", ctx, fp64_tf=fp64))
    torch.cuda.empty_cache()
    attempt("config1", lambda: config1_line(cp, ctx, args.steps))
    attempt("config0_aligned", lambda: aligned("config0", ctx, 20, fp64))
    attempt("config2_aligned", lambda: aligned("config2", ctx, 10, fp64))
    attempt("cpu_baselines", lambda: cpu_baselines(orc.max_threads()))
    return sec
