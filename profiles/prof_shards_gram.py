"""Config 4 in 8 shards: the row-Gram build (first application of the GRAM operator) of every shard
timed alone, for the q-pass-time cut (default) and the plan-entries cut (CPHIFI_OBS_SHARD_BY_ENTRIES)."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25691_b200 as cp  # noqa: E402
from inputs import configs  # noqa: E402
from paper_2603_25691_b200 import _capi  # noqa: E402

lib = _capi.load()
ctx = cp.Context(0)
dev = torch.device("cuda", 0)
cfg = configs.config4()
n, r, q = cfg.shape[0], cfg.r, cfg.q
idx, vals = cp.synth_observations_device(cfg, ctx)
mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
x = torch.randn(n * r, dtype=torch.float64, device=dev)
y = torch.empty_like(x)
out = {}
for S in (1, 8):
    for by_entries in ((False,) if S == 1 else (False, True)):
        rows = []
        for s in range(S):
            obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), q, keepalive=(idx, vals),
                                        coalesce=cfg.coalesce)
            obs.shard_by_entries = by_entries
            p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho, shard=s, shards=S)
            p.set_operator("gram")
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            for _ in range(3):
                _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
            torch.cuda.synchronize()
            stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(20):
                    _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
                e1.record(stream)
            torch.cuda.synchronize()
            apply_ms = e0.elapsed_time(e1) / 20
            qt, ql = ctypes.c_int64(), ctypes.c_int64()
            _capi.check(lib.cphifi_obs_info(obs.plan(0, ctx, s, S).h, ctypes.byref(qt), ctypes.byref(ql), None))
            rows.append(dict(shard=s, build_ms=(t1 - t0) * 1e3, entries=ql.value, gram_apply_ms=apply_ms))
            del p, obs
            torch.cuda.empty_cache()
        key = f"S{S}_{'entries' if by_entries else 'time'}"
        out[key] = dict(max_ms=max(rw["build_ms"] for rw in rows), shards=rows)
        out[key]["max_apply_ms"] = max(rw["gram_apply_ms"] for rw in rows)
        print(key, "max %.2f ms" % out[key]["max_ms"], ["%.1f" % rw["build_ms"] for rw in rows],
              "gram application ms", ["%.3f" % rw["gram_apply_ms"] for rw in rows], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/shard_gram_config4.json", "w"), indent=1)
