"""Config 4 cut into S observation shards, every shard's operator application timed ALONE on one GPU
(one shard at a time: no rank waits on another), for the equal-count cut and the cost-balanced cut
(capi.cu balanced_shard_cut).  The slowest shard bounds the N-GPU application (plus the n x r
all-reduce, not timed here): projected strong scaling = t(S = 1) / max_s t(s)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25691_b200 as cp  # noqa: E402
from inputs import configs  # noqa: E402
from paper_2603_25691_b200 import _capi  # noqa: E402


def main():
    lib = _capi.load()
    ctx = cp.Context(0)
    dev = torch.device("cuda", 0)
    cfg = configs.config4() if len(sys.argv) < 2 or sys.argv[1] == "4" else configs.config3()
    n, r, q = cfg.shape[0], cfg.r, cfg.q
    idx, vals = cp.synth_observations_device(cfg, ctx)
    torch.cuda.synchronize()
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
    x = torch.randn(n * r, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    out = {"config": cfg.name if hasattr(cfg, "name") else "config", "q": q, "cuts": {}}
    for S in (1, 2, 4, 8):
        for equal in ((0,) if S == 1 else (1, 0)):
            os.environ["CPHIFI_SHARD_EQUAL_COUNT"] = str(equal)
            rows = []
            ysum = torch.zeros_like(x)
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
                    for _ in range(10):
                        _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
                    e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 10
                ms6 = (ctypes.c_double * 6)()
                _capi.check(lib.cphifi_unaligned_matvec_timed(p.handle, x.data_ptr(), y.data_ptr(), 5, ms6))
                qp = p.qpass_plan()
                qt, ql = ctypes.c_int64(), ctypes.c_int64()
                _capi.check(lib.cphifi_obs_info(obs.plan(0, ctx, s, S).h, ctypes.byref(qt), ctypes.byref(ql), None))
                rows.append(dict(shard=s, ms=ms, entries=ql.value, dense_rows=qp["dense_rows"],
                                 sparse_entries=qp["sparse_entries"], runs_ms=ms6[1], dense_ms=ms6[2],
                                 gemm_ms=ms6[0] + ms6[4]))
                ysum += y  # row-sharded operator without a communicator: y = this shard's partial y_s
                del p, obs
                torch.cuda.empty_cache()
            key = f"S{S}_{'equal' if equal else 'balanced'}"
            tmax = max(rw["ms"] for rw in rows)
            out["cuts"][key] = dict(max_ms=tmax, sum_ms=sum(rw["ms"] for rw in rows), shards=rows)
            if S == 1:
                yref = ysum.clone()
                out["t1_ms"] = tmax
            else:
                out["cuts"][key]["projected_speedup"] = out["t1_ms"] / tmax
                out["cuts"][key]["sum_of_partials_rel_err"] = float(torch.linalg.norm(ysum - yref) / torch.linalg.norm(yref))
            print(key, "max %.3f ms" % tmax, ["%.2f" % rw["ms"] for rw in rows],
                  out["cuts"][key].get("sum_of_partials_rel_err"), flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/shard_cuts_config4.json", "w"), indent=1)


if __name__ == "__main__":
    main()
