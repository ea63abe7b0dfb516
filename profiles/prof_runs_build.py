import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_25691_b200 as cp
from inputs import configs
ctx = cp.Context(0)
cfg = configs.config4()
n, r = cfg.shape[0], cfg.r
idx, vals = cp.synth_observations_device(cfg, ctx)
mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), cfg.q, keepalive=(idx, vals), coalesce=cfg.coalesce)
model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
for it in range(2):
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho)
    p.set_operator("stream")
    t0 = time.perf_counter(); pl = p.qpass_plan(); print("qpass plan", time.perf_counter() - t0, pl, flush=True)
    del p
