"""Configs 3 / 4 at full size: setup (device generation, sort/CSR plan, B, V) and operator
applications timed with CUDA events on the library stream (inputs are far larger than L2, so no
flush is needed), the per-CTA phase trace, and size-independent checks (symmetry x'Ay = y'Ax and
linearity of the operator).

  python profiles/prof_large.py --config 3 [--q 200000000] [--iters 5]
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2603_25691_b200 as cp
from paper_2603_25691_b200 import _capi
from inputs import configs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--q", type=int, default=0)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--trace", type=int, default=1)
    ap.add_argument("--solve", type=int, default=0)
    ap.add_argument("--coalesce", type=int, default=0)
    args = ap.parse_args()
    cfg = configs.config3() if args.config == 3 else configs.config4()
    q = args.q or cfg.q
    n, r, d = cfg.shape[0], cfg.r, len(cfg.shape)
    ctx = cp.Context(0)
    lib = _capi.load()
    out = {"config": cfg.name, "q": q, "n": n, "r": r, "d": d}
    t0 = time.perf_counter()
    idx, vals = cp.synth_observations_device(cfg, ctx, q)
    torch.cuda.synchronize()
    out["gen_s"] = time.perf_counter() - t0
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), q, keepalive=(idx, vals),
                                coalesce=bool(args.coalesce))
    model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
    t0 = time.perf_counter()
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho)
    out["plan_s"] = time.perf_counter() - t0
    qt, ql = ctypes.c_int64(), ctypes.c_int64()
    _capi.check(lib.cphifi_obs_info(obs.plan(0, ctx).h, ctypes.byref(qt), ctypes.byref(ql), None))
    out["coalesce"] = bool(args.coalesce)
    out["plan_entries"] = ql.value
    del idx, vals
    obs.release_inputs()
    torch.cuda.empty_cache()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    gen = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(n * r, dtype=torch.float64, device=dev, generator=gen)
    y = torch.empty_like(x)
    for _ in range(2):
        _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
    ts = []
    for _ in range(args.iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
            b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    ms6 = (ctypes.c_double * 6)()
    _capi.check(lib.cphifi_unaligned_matvec_timed(p.handle, x.data_ptr(), y.data_ptr(), max(1, args.iters // 2), ms6))
    hbm = 6452.2
    b_alg = 4 * d * q + 16 * n * n + 48 * n * r
    f_alg = (d + 2) * r * q + 4 * n * n * r
    out.update({"matvec_ms": ms, "matvecs_per_s": 1e3 / ms, "phase_ms": list(ms6),
                "alg_bytes": b_alg, "alg_flops": f_alg, "hbm_frac": b_alg / (ms / 1e3) / 1e9 / hbm,
                "fp64_tflops": f_alg / (ms / 1e3) / 1e12,
                "k1_hbm_frac": (4 * d * q + 16 * n * r) / (ms6[1] / 1e3) / 1e9 / hbm})
    # size-independent properties: symmetry and linearity of the operator
    z = torch.randn(n * r, dtype=torch.float64, device=dev, generator=gen)
    az = torch.empty_like(z)
    _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, z.data_ptr(), az.data_ptr()))
    xs = torch.empty_like(x)
    xs.copy_(x + 2.5 * z)
    axs = torch.empty_like(x)
    _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, xs.data_ptr(), axs.data_ptr()))
    ctx.synchronize()
    sym = abs(float(z @ y) - float(x @ az)) / abs(float(z @ y))
    lin = float(torch.linalg.norm(axs - (y + 2.5 * az)) / torch.linalg.norm(axs))
    out.update({"symmetry_rel": sym, "linearity_rel": lin})
    # row-Gram operator: one-time build, then applications
    _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))  # streaming A x
    ctx.synchronize()
    t0 = time.perf_counter()
    p.set_operator("gram")
    ytmp = torch.empty_like(y)
    _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), ytmp.data_ptr()))
    ctx.synchronize()
    out["gram_build_plus_first_s"] = time.perf_counter() - t0
    yg = torch.empty_like(y)
    ts = []
    for _ in range(max(3, args.iters)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), yg.data_ptr()))
            b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out["gram_matvec_ms"] = float(np.median(ts))
    out["gram_vs_stream_rel"] = float(torch.linalg.norm(yg - y) / torch.linalg.norm(y))
    if args.solve:
        t0 = time.perf_counter()
        mode.eig() if hasattr(mode, "eig") else None
        out["eigK_s"] = time.perf_counter() - t0
        rep = cp.SolveReport()
        cp.solve_unaligned_pcg(p, cp.PcgConfig(cfg.tol, cfg.max_iter, True), rep)
        out["pcg_gram"] = {"iterations": rep.iterations, "relative_residual": rep.relative_residual,
                           "converged": rep.converged, "wall_s": rep.wall_time_s, "setup_s": rep.setup_s,
                           "history_tail": rep.residual_history[-3:]}
        p.set_operator("stream")
    p.set_operator("stream")
    if args.trace:
        cap = 8 * 4096
        st = np.zeros(cap, dtype=np.uint64)
        ctas = ctypes.c_int()
        _capi.check(lib.cphifi_unaligned_matvec_trace(p.handle, x.data_ptr(), y.data_ptr(),
                                                      st.ctypes.data_as(_capi.c_uint64_p), cap, ctypes.byref(ctas)))
        s = st[: 8 * ctas.value].reshape(ctas.value, 8).astype(np.float64)
        t0 = s[:, 0].min()
        names = ["entry", "AL done", "tile0 rdy", "B loop", "B done", "barrier", "-", "exit"]
        tr = {}
        for k, nm in enumerate(names):
            col = s[:, k]
            col = col[col > 0]
            if col.size:
                col = (col - t0) / 1e3
                tr[nm] = [round(float(col.min()), 2), round(float(np.median(col)), 2), round(float(col.max()), 2)]
        out["trace_us_min_med_max"] = tr
        out["ctas"] = ctas.value
    print(json.dumps(out))


if __name__ == "__main__":
    main()
