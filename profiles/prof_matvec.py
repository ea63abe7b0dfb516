"""Short, ncu-friendly driver: config-1 (or another config) operator applications only.

  python profiles/prof_matvec.py [--config 1] [--iters 20] [--flush 1]
Prints per-application device times (CUDA events on the library stream) with and without an
L2 flush before each application.  Used for the `ncu --set full` captures under profiles/.
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2603_25691_b200 as cp
from paper_2603_25691_b200 import _capi
from inputs import configs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--flush", type=int, default=1)
    args = ap.parse_args()
    c = configs.config1() if args.config == 1 else configs.small_unaligned()
    n, r = c.shape[0], c.r
    ctx = cp.Context(0)
    mode = cp.RkhsMode(c.points, c.ell, c.lam, ctx=ctx)
    obs = cp.ObservationSet(c.shape, c.idx, c.vals, multiset=True)
    p = cp.make_unaligned_subproblem(obs, cp.KruskalModel([np.zeros((n, r))] + c.factors[1:]), 0, mode, c.rho)
    dev = torch.device("cuda", 0)
    x = torch.randn(n * r, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    lib = _capi.load()
    for flush_on in ([1, 0] if args.flush else [0]):
        ts = []
        for i in range(args.iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                if flush_on:
                    flush.add_(1)
                a.record(stream)
                _capi.check(lib.cphifi_unaligned_matvec_device(p.handle, x.data_ptr(), y.data_ptr()))
                b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts = np.array(ts[3:])
        print(f"flush={flush_on}: median {np.median(ts):.2f} us  min {ts.min():.2f} us  (n={ts.size})")
    # per-CTA phase stamps (%globaltimer, ns): when did the slowest / fastest CTA reach each point
    names = ["entry", "AL done", "tile0 rdy", "B loop", "B done", "barrier", "-", "exit"]
    cap = 8 * 4096
    st = np.zeros(cap, dtype=np.uint64)
    ctas = ctypes.c_int()
    for rep in range(3):
        with torch.cuda.stream(stream):
            flush.add_(1)
        stream.synchronize()
        _capi.check(lib.cphifi_unaligned_matvec_trace(p.handle, x.data_ptr(), y.data_ptr(),
                                                      st.ctypes.data_as(_capi.c_uint64_p), cap, ctypes.byref(ctas)))
    s = st[: 8 * ctas.value].reshape(ctas.value, 8).astype(np.float64)
    t0 = s[:, 0].min()
    print(f"trace over {ctas.value} CTAs (us from first entry): phase point: min / median / max")
    for k, nm in enumerate(names):
        col = s[:, k]
        col = col[col > 0]
        if col.size:
            col = (col - t0) / 1e3
            print(f"  {nm:9s} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}")


if __name__ == "__main__":
    main()
