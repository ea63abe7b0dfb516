"""Per-phase device times of the config-1 operator (cphifi_unaligned_matvec_timed, L2 flushed
before each application): K X GEMM / scatter-gather / all-reduce / y GEMM (or the fused kernel)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_25691_b200 as cp  # noqa: E402
from paper_2603_25691_b200 import _capi  # noqa: E402
from inputs import configs

c = configs.config1()
n, r = c.shape[0], c.r
ctx = cp.Context(0)
mode = cp.RkhsMode(c.points, c.ell, c.lam, ctx=ctx)
p = cp.make_unaligned_subproblem(cp.ObservationSet(c.shape, c.idx, c.vals),
                                 cp.KruskalModel([np.zeros((n, r))] + c.factors[1:]), 0, mode, c.rho)
dev = torch.device("cuda", 0)
x = torch.randn(n * r, dtype=torch.float64, device=dev)
y = torch.empty_like(x)
stream = torch.cuda.ExternalStream(ctx.stream(), device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
lib = _capi.load()
ms6 = (ctypes.c_double * 6)()
acc = np.zeros(6)
for it in range(60):
    with torch.cuda.stream(stream):
        flush.add_(1)
    _capi.check(lib.cphifi_unaligned_matvec_timed(p.handle, x.data_ptr(), y.data_ptr(), 1, ms6))
    if it >= 10:
        acc += np.array(ms6[:])
acc /= 50
print("phases us (xhat, B, -, allreduce, y, total):", np.round(acc * 1e3, 2))
