"""The stream operator (k_stream.cu) at full config 3 / 4: per-application device time of the
scatter-gather kernel(s) with CUDA events, for variants selected by environment variables
(CPHIFI_STREAM_PARTS, ...), plus a parity check of every variant against the first one
(same plan, same x: relative difference of y).  Inputs far exceed L2 (no flush needed).

  python profiles/prof_stream.py --config 4 [--iters 10] [--variants "CPHIFI_STREAM_PARTS=0;"]
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_25691_b200 as cp  # noqa: E402
from inputs import configs  # noqa: E402
from paper_2603_25691_b200 import _capi  # noqa: E402


def build(cfg, ctx, q):
    idx, vals = cp.synth_observations_device(cfg, ctx, q)
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), q, keepalive=(idx, vals),
                                coalesce=cfg.coalesce)
    n, r = cfg.shape[0], cfg.r
    model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
    return obs, mode, model


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--q", type=int, default=0)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--variants", default="")
    args = ap.parse_args()
    cfg = configs.config3() if args.config == 3 else configs.config4()
    q = args.q or cfg.q
    n, r = cfg.shape[0], cfg.r
    ctx = cp.Context(0)
    lib = _capi.load()
    obs, mode, model = build(cfg, ctx, q)
    dev = torch.device("cuda", 0)
    x = torch.randn(n * r, dtype=torch.float64, device=dev, generator=torch.Generator(device=dev).manual_seed(0))
    y = torch.empty_like(x)
    out = {"config": cfg.name, "q": q, "variants": []}
    y_ref = None
    for var in [""] + [v for v in args.variants.split(";") if v.strip()]:
        env = dict(kv.split("=") for kv in var.split(",") if kv.strip())
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        t0 = time.perf_counter()
        p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho)
        plan_s = time.perf_counter() - t0
        p.set_operator("stream")
        ms6 = (ctypes.c_double * 6)()
        _capi.check(lib.cphifi_unaligned_matvec_timed(p.handle, x.data_ptr(), y.data_ptr(), 2, ms6))
        _capi.check(lib.cphifi_unaligned_matvec_timed(p.handle, x.data_ptr(), y.data_ptr(), args.iters, ms6))
        torch.cuda.synchronize()
        yy = y.clone()
        rel = None if y_ref is None else float(torch.linalg.norm(yy - y_ref) / torch.linalg.norm(y_ref))
        if y_ref is None:
            y_ref = yy
        out["variants"].append({"env": env, "plan_s": plan_s, "stream_ms": ms6[1], "app_ms": ms6[5],
                                "rel_vs_first": rel, "qpass_plan": p.qpass_plan(),
                                "y_sum": float(yy.sum()), "y_norm": float(torch.linalg.norm(yy))})
        print(json.dumps(out["variants"][-1]), flush=True)
        del p
        torch.cuda.empty_cache()
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    print(json.dumps(out))


if __name__ == "__main__":
    main()
