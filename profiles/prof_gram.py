"""Row-Gram build time at full config 3 / 4 size: FMA build vs DMMA build (CPHIFI_GRAM_DMMA)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_25691_b200 as cp  # noqa: E402
from inputs import configs  # noqa: E402

ctx = cp.Context(0)
for which in sys.argv[1:] or ["config3"]:
    cfg = getattr(configs, which)()
    n, r = cfg.shape[0], cfg.r
    idx, vals = cp.synth_observations_device(cfg, ctx)
    torch.cuda.synchronize()
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), cfg.q, keepalive=(idx, vals),
                                coalesce=cfg.coalesce)
    model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
    from paper_2603_25691_b200 import _capi
    lib = _capi.load()
    xd = torch.randn(n * r, dtype=torch.float64, device="cuda")
    yd = torch.empty_like(xd)
    ys = {}
    for dm in ("0", "1"):
        os.environ["CPHIFI_GRAM_DMMA"] = dm
        p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho)
        p.set_operator("gram")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, xd.data_ptr(), yd.data_ptr()))  # builds G
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ys[dm] = yd.cpu().numpy()
        _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, xd.data_ptr(), yd.data_ptr()))
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{which} dmma={dm}: build+apply {1e3 * (t1 - t0):.1f} ms, apply {1e3 * (t2 - t1):.2f} ms")
        del p
    print(f"{which} G-operator rel diff dmma vs fma {np.linalg.norm(ys['0'] - ys['1']) / np.linalg.norm(ys['0']):.2e}")
