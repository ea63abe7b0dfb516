"""Full-size parity evidence: config 3 (q = 2e8 draws, 4-way, Matern-3/2) solved by
the device PCG and by the oracle's streaming restatement (multithreaded C, multiset semantics)
on the SAME seeded inputs and the same eig(K): iteration counts, final residuals,
the relative residual history and W.  Optionally config 4 (q = 1e9 draws): the first
`--iters4` PCG iterations' residual history (the oracle needs ~1 min per operator application).

  python profiles/parity_full.py [--config4 0] [--iters4 2] > out.json
"""
import argparse
import json
import os
import sys
import time
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_25691_b200 as cp  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from inputs import configs  # noqa: E402


def run(which, ctx, max_iter, tol):
    cfg = getattr(configs, which)()
    n, r = cfg.shape[0], cfg.r
    idx_d, vals_d = cp.synth_observations_device(cfg, ctx)
    torch.cuda.synchronize()
    idx = idx_d.cpu().numpy().reshape(len(cfg.shape), -1)
    vals = vals_d.cpu().numpy().reshape(-1)
    kern_fn = orc.matern32_kernel if cfg.kernel == "matern32" else orc.gaussian_kernel
    kern = kern_fn(cfg.points, cfg.ell)
    t0 = time.perf_counter()
    ek = orc.sym_eig(kern)
    eig_s = time.perf_counter() - t0
    factors = [np.zeros((n, r))] + cfg.factors[1:]
    # device: same inputs, same eig(K); plan without coalescing (raw draws, multiset)
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    mode.set_eig(ek.u, ek.d)
    obs = cp.DeviceObservations(cfg.shape, idx_d.data_ptr(), vals_d.data_ptr(), cfg.q, keepalive=(idx_d, vals_d),
                                coalesce=False)
    p = cp.make_unaligned_subproblem(obs, cp.KruskalModel(factors), 0, mode, cfg.rho)
    p.set_operator("gram")
    rep = cp.SolveReport()
    t0 = time.perf_counter()
    w = cp.solve_unaligned_pcg(p, cp.PcgConfig(tol, max_iter, record_history=True), rep)
    gpu_s = time.perf_counter() - t0
    b_dev = p.b
    v_dev = p.v
    del p, obs, idx_d, vals_d
    torch.cuda.empty_cache()
    # oracle: streaming restatement, all host threads
    th = orc.max_threads()
    t0 = time.perf_counter()
    b = orc.sampled_mttkrp_stream(cfg.shape, 0, idx, vals, factors, n, threads=th)
    v = orc.gram_khatri_rao(factors, 0)
    ev = orc.sym_eig(v)
    sub = SimpleNamespace(n=n, r=r, density=cfg.q / float(np.prod(np.array(cfg.shape, dtype=np.float64))),
                          lam=cfg.lam, rho=cfg.rho, v=v)
    m_inv = orc.build_preconditioner(sub, ek, ev)
    rhs = orc.gemm(kern, b, threads=th).reshape(-1, order="F")
    nmv = [0]

    def apply_a(x):
        nmv[0] += 1
        return orc.unaligned_matvec_stream(cfg.shape, 0, idx, factors, kern, cfg.lam, cfg.rho, x, threads=th)

    orep = orc.SolveReport()
    wo = orc.pcg(apply_a, lambda x: m_inv.apply(x, th), rhs, orc.PcgConfig(tol, max_iter, record_history=True),
                 orep).reshape((n, r), order="F")
    cpu_s = time.perf_counter() - t0
    hist = list(rep.residual_history)
    ohist = list(orep.residual_history)
    k = min(len(hist), len(ohist))
    return {
        "config": which, "q": cfg.q, "n": n, "r": r, "tol": tol, "max_iter": max_iter,
        "gpu": {"iterations": rep.iterations, "relative_residual": rep.relative_residual, "wall_s": gpu_s},
        "oracle": {"iterations": orep.iterations, "relative_residual": orep.relative_residual, "wall_s": cpu_s,
                   "threads": th, "operator_applications": nmv[0]},
        "iterations_within_1": abs(rep.iterations - orep.iterations) <= 1,
        "B_rel_diff": float(np.linalg.norm(b_dev - b) / np.linalg.norm(b)),
        "V_rel_diff": float(np.linalg.norm(v_dev - v) / np.linalg.norm(v)),
        "W_rel_diff": float(np.linalg.norm(w - wo) / np.linalg.norm(wo)),
        "history_gpu": hist, "history_oracle": ohist,
        "history_max_rel_diff": float(max(abs(a - b) / b for a, b in zip(hist[:k], ohist[:k]))) if k else None,
        "eigK_s": eig_s,
        "note": "device PCG: row-Gram operator, eigenbasis PCG (large n); oracle: streaming operator, "
                "reference PCG recurrence, same eig(K)",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config4", type=int, default=0)
    ap.add_argument("--iters4", type=int, default=2)
    args = ap.parse_args()
    ctx = cp.Context(0)
    out = {"config3": run("config3", ctx, 500, 1e-8)}
    if args.config4:
        out["config4_first_iterations"] = run("config4", ctx, args.iters4, 1e-30)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
