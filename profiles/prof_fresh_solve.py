"""Config-4 fresh-factor PCG solve (a new subproblem on the same observation plan: B, V, G build,
eig(V), preconditioner, PCG) with the setup phases timed (CPHIFI_SOLVE_TIMING / CPHIFI_GRAM_TIMING
print them to stderr).  Run once per build variant (CPHIFI_GRAM3_PARTS=0 / default).
  python profiles/prof_fresh_solve.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_25691_b200 as cp  # noqa: E402
from inputs import configs  # noqa: E402

cfg = configs.config4()
ctx = cp.Context(0)
n, r = cfg.shape[0], cfg.r
idx, vals = cp.synth_observations_device(cfg, ctx)
mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), cfg.q, keepalive=(idx, vals),
                            coalesce=cfg.coalesce)
model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho)
p.set_operator("stream")
p.qpass_plan()  # the q-pass plan (shared by every subproblem on these observations)
torch.cuda.synchronize()
pc = cp.PcgConfig(cfg.tol, cfg.max_iter)
g = np.random.default_rng(5)
for rep_i in range(3):
    fac = [np.zeros((n, r))] + [f * (1.0 + 0.01 * g.normal(size=f.shape)) for f in cfg.factors[1:]]
    t0 = time.perf_counter()
    p2 = cp.make_unaligned_subproblem(obs, cp.KruskalModel(fac), 0, mode, cfg.rho)
    t_sub = time.perf_counter() - t0
    rep = cp.SolveReport()
    cp.solve_unaligned_pcg(p2, pc, rep)
    print(json.dumps({"rep": rep_i, "subproblem_s": t_sub, "pcg_wall_s": rep.wall_time_s, "setup_s": rep.setup_s,
                      "iterations": rep.iterations}), flush=True)
    del p2
