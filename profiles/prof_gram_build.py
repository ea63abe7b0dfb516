"""Row-Gram build cost at full size (configs 3 / 4): host-timed first gram application (build +
apply) on two fresh plans of the same observation set, so the second excludes one-time costs
(function attributes, first allocations).  Under `ncu --metrics gpu__time_duration.sum` the
launch list gives the build kernel's device time alone.
  python profiles/prof_gram_build.py config3 config4"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_25691_b200 as cp  # noqa: E402
from paper_2603_25691_b200 import _capi  # noqa: E402
from inputs import configs

ctx = cp.Context(0)
lib = _capi.load()
for which in sys.argv[1:] or ["config3"]:
    cfg = getattr(configs, which)()
    n, r = cfg.shape[0], cfg.r
    idx, vals = cp.synth_observations_device(cfg, ctx)
    torch.cuda.synchronize()
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), cfg.q, keepalive=(idx, vals),
                                coalesce=cfg.coalesce)
    model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
    xd = torch.randn(n * r, dtype=torch.float64, device="cuda")
    yd = torch.empty_like(xd)
    for rep in range(2):
        p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho)
        p.set_operator("gram")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, xd.data_ptr(), yd.data_ptr()))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, xd.data_ptr(), yd.data_ptr()))
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{which} plan {rep}: build+apply {1e3 * (t1 - t0):.2f} ms, apply {1e3 * (t2 - t1):.3f} ms", flush=True)
        del p
    del obs, idx, vals
    torch.cuda.empty_cache()
