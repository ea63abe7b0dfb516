import os, sys, time, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2603_25691_b200 as cp
from paper_2603_25691_b200 import _capi
from inputs import configs
ctx = cp.Context(0)
cfg = configs.config4()
n, r = cfg.shape[0], cfg.r
idx, vals = cp.synth_observations_device(cfg, ctx)
mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), cfg.q, keepalive=(idx, vals), coalesce=cfg.coalesce)
model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
t0 = time.perf_counter(); p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho); print("create", time.perf_counter() - t0, p.operator(), flush=True)
t0 = time.perf_counter(); mode.eig(); print("eigK", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter(); cp.build_preconditioner(p); print("precond", time.perf_counter() - t0, flush=True)
x = np.random.default_rng(0).normal(size=n * r)
t0 = time.perf_counter(); cp.unaligned_matvec(p, x); print("first gram matvec (G build)", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter(); cp.unaligned_matvec(p, x); print("second gram matvec", time.perf_counter() - t0, flush=True)
rep = cp.SolveReport()
t0 = time.perf_counter(); cp.solve_unaligned_pcg(p, cp.PcgConfig(cfg.tol, cfg.max_iter), rep); print("solve", time.perf_counter() - t0, rep.setup_s, rep.iterations, flush=True)
rep = cp.SolveReport()
t0 = time.perf_counter(); cp.solve_unaligned_pcg(p, cp.PcgConfig(cfg.tol, cfg.max_iter), rep); print("solve2", time.perf_counter() - t0, rep.setup_s, rep.iterations, flush=True)
# the bench's order: stream-operator solves first (run tables built), then the row-Gram solve on a
# fresh plan of the same observations
p.set_operator("stream")
rep = cp.SolveReport()
t0 = time.perf_counter(); cp.solve_unaligned_pcg(p, cp.PcgConfig(cfg.tol, cfg.max_iter), rep); print("stream solve", time.perf_counter() - t0, rep.setup_s, flush=True)
t0 = time.perf_counter(); p3 = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho); print("create p3", time.perf_counter() - t0, flush=True)
rep = cp.SolveReport()
t0 = time.perf_counter(); cp.solve_unaligned_pcg(p3, cp.PcgConfig(cfg.tol, cfg.max_iter), rep); print("gram solve p3", time.perf_counter() - t0, rep.setup_s, flush=True)
