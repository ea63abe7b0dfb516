"""Secondary measurements reported inside bench.py's JSON line (N = 1 only).

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
    from paper_2603_25691_b200 import _capi, configs
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


def config1_pcg(cp, p, c):
    """Full device PCG solves of config 1 with both operator forms (wall clock, host loop)."""
    out = {}
    for op in ("stream", "gram"):
        p.set_operator(op)
        rep = cp.SolveReport()
        t0 = time.perf_counter()
        cp.solve_unaligned_pcg(p, cp.PcgConfig(c.tol, c.max_iter), rep)  # first: includes G build for gram
        first = time.perf_counter() - t0
        rep = cp.SolveReport()
        cp.solve_unaligned_pcg(p, cp.PcgConfig(c.tol, c.max_iter), rep)
        out[op] = {"iterations": rep.iterations, "relative_residual": rep.relative_residual, "wall_s": rep.wall_time_s,
                   "first_call_s": first, "matvecs": rep.matvecs}
    p.set_operator("stream")
    return out


def gram_matvec_ms(p, lib, x, y, stream, flush, steps=50):
    import torch
    from paper_2603_25691_b200 import _capi
    p.set_operator("gram")
    _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))  # builds G
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.add_(1)
            a.record(stream)
            _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
            b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    p.set_operator("stream")
    return float(np.median(ts))


def large(which, ctx, iters=3, solve=True, fp64_tf=None):
    """Configs 3/4 at full size: per-observation operator, row-Gram operator, PCG (row-Gram).
    Config 4's plan coalesces repeated draws (cfg.coalesce): the streamed entries are the distinct
    multi-indices, the algorithmic bytes / flops below stay those of the as-given q draws."""
    import torch

    import paper_2603_25691_b200 as cp
    from paper_2603_25691_b200 import _capi, configs
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


def als_updates(ctx, p, c):
    """ALS infinite-mode update on device: config 1 (unaligned, PCG warm-started
    from the previous W as AlsState does) and config 2 (aligned decoupled), wall clock per update
    plus the device-timed split (solve / factor update + error terms)."""
    import paper_2603_25691_b200 as cp
    from inputs import configs
    out = {}
    cfg = cp.PcgConfig(c.tol, c.max_iter)
    u = cp.update_infinite_mode_unaligned(p, cfg)
    t0 = time.perf_counter()
    u2 = cp.update_infinite_mode_unaligned(p, cfg, warm_start=u.w)
    out["config1_unaligned"] = {"wall_s_warm": time.perf_counter() - t0, "relative_error": u.relative_error,
                                "iterations_cold": u.report.iterations, "iterations_warm": u2.report.iterations,
                                "solve_s": u.solve_s, "update_and_error_s": u.update_s}
    # a whole unaligned ALS sweep on device (mode 0 infinite, modes 1, 2 finite, then the error)
    st = cp.UnalignedAlsState(cp.ObservationSet(c.shape, c.idx, c.vals), p.mode,
                              cp.KruskalModel([np.zeros((c.shape[0], c.r))] + c.factors[1:]), rho=c.rho, inner=cfg)
    its = [st.sweep() for _ in range(4)]  # the first sweep builds the per-mode plans
    out["config1_unaligned_sweep"] = {"wall_s_per_sweep": float(np.median([it.wall_time_s for it in its[1:]])),
                                      "first_sweep_s": its[0].wall_time_s,
                                      "rel_errors": [it.rel_error for it in its],
                                      "pcg_iterations": [it.pcg_iterations for it in its],
                                      "note": "infinite mode: PCG warm-started + A_0 = K W; finite modes: row "
                                              "least squares (row Grams + batched Jacobi pseudo-inverse); error pass"}
    c2 = configs.config2()
    n, r = c2.shape[0], c2.r
    mode = cp.RkhsMode(c2.points, c2.ell, c2.lam, ctx=ctx)
    t = cp.DenseTensor(c2.shape, c2.tensor)
    model = cp.KruskalModel([np.zeros((n, r))] + c2.factors[1:])
    cp.update_infinite_mode_aligned(t, model, 0, mode)  # eig(K), tensor upload, ||T||^2 once
    t0 = time.perf_counter()
    ua = cp.update_infinite_mode_aligned(t, model, 0, mode)
    # whole aligned sweeps on device (mode 0 infinite; modes 1, 2 finite: A_k = B_k V_k^+)
    g = np.random.default_rng(0)
    init = [np.zeros((n, r))] + [g.normal(size=(s_, r)) for s_ in c2.shape[1:]]
    st = cp.AlignedAlsState(t, mode, cp.KruskalModel(init))
    its = [st.sweep() for _ in range(4)]
    out["config2_aligned_sweep"] = {"wall_s_per_sweep": float(np.median([it.wall_time_s for it in its[1:]])),
                                    "rel_errors": [it.rel_error for it in its],
                                    "note": "MTTKRP for modes 0, 1, 2 on the TMA DMMA ring (k > 0: transposed "
                                            "unfolding tiles), decoupled solve, B V^+ finite updates, Gram-identity "
                                            "errors"}
    out["config2_aligned"] = {"wall_s": time.perf_counter() - t0, "relative_error": ua.relative_error,
                              "aligned_residual": ua.residual, "solve_s": ua.solve_s,
                              "update_and_error_s": ua.update_s,
                              "note": "relative error via ||T||^2 - 2<A,B> + 1'(A'A o V)1: no N-sized pass"}
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
