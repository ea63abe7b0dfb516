"""Row-Gram build variants at full config 4 (or 3): host-timed build (first gram application minus a
repeat application) for the default build and the register-fragment build over the q-pass plan's
factor-block parts (CPHIFI_GRAM3_PARTS=1: mode 0 through L1 per entry; =3: mode 0 hoisted per run),
each checked against the stream operator on the same x (relative difference of y).
  python profiles/prof_gram_parts.py [config4] [variants, e.g. "0 1 3"]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_25691_b200 as cp  # noqa: E402
from paper_2603_25691_b200 import _capi  # noqa: E402
from inputs import configs  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "config4"
variants = (sys.argv[2] if len(sys.argv) > 2 else "0 1 3").split()
ctx = cp.Context(0)
lib = _capi.load()
cfg = getattr(configs, which)()
n, r = cfg.shape[0], cfg.r
idx, vals = cp.synth_observations_device(cfg, ctx)
torch.cuda.synchronize()
mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), cfg.q, keepalive=(idx, vals),
                            coalesce=cfg.coalesce)
model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
xd = torch.randn(n * r, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(0))
yd = torch.empty_like(xd)
p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho)
p.set_operator("stream")
_capi.check(lib.cphifi_unaligned_matvec_device(p.handle, xd.data_ptr(), yd.data_ptr()))
torch.cuda.synchronize()
y_ref = yd.clone()
del p
for v in variants:
    if v == "0":
        os.environ.pop("CPHIFI_GRAM3_PARTS", None)
    else:
        os.environ["CPHIFI_GRAM3_PARTS"] = v
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
        rel = float(torch.linalg.norm(yd - y_ref) / torch.linalg.norm(y_ref))
        print(json.dumps({"config": which, "variant": v, "rep": rep, "build_ms": 1e3 * ((t1 - t0) - (t2 - t1)),
                          "apply_ms": 1e3 * (t2 - t1), "rel_vs_stream": rel}), flush=True)
        del p
