"""ncu driver: config-2 aligned solve (MTTKRP + Gram + decoupled), a few repetitions."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_secondary as bs  # noqa: E402
import paper_2603_25691_b200 as cp  # noqa: E402

ctx = cp.Context(0)
o = bs.aligned(sys.argv[1] if len(sys.argv) > 1 else "config2", ctx, 2, 37.0)
print({k: o[k] for k in ("solve_ms", "mttkrp_ms", "decoupled_ms")})
