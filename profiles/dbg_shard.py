"""Stress of the sharded plans on the skewed multiset of tests/test_gpu_multirank.py (developer)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_25691_b200 as cp  # noqa: E402
from tests.test_gpu_multirank import _skewed_case  # noqa: E402

ctx = cp.Context(0)
for rep in range(int(os.environ.get("REPS", "3"))):
    for d3 in (True, False):
        shape, r, idx, vals, pts, factors = _skewed_case(d3)
        n = shape[0]
        mode = cp.RkhsMode(pts, 0.05, 1e-3, ctx=ctx)
        model = cp.KruskalModel([np.zeros((n, r))] + factors[1:])
        x = np.random.default_rng(3).normal(size=n * r)
        for coalesce in (True, False):
            for S in (2, 3, 8):
                for eq in (False, True):
                    obs = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
                    obs.equal_count_shards = eq
                    for s in range(S):
                        print(rep, d3, coalesce, S, eq, s, flush=True)
                        p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6, shard=s, shards=S)
                        p.set_operator("stream")
                        y = cp.unaligned_matvec(p, x)
                        assert np.all(np.isfinite(y))
print("stress ok")
