"""Config 3 stream-operator application time (developer: CPHIFI_RUNS_VAR A/B)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_secondary as bs  # noqa: E402
import paper_2603_25691_b200 as cp  # noqa: E402

ctx = cp.Context(0)
out = bs.large("config3", ctx, iters=5, solve=False)
print({k: v for k, v in out.items() if "ms" in k or "stream" in k})
