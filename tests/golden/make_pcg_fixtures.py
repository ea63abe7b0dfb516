"""Full-size PCG fixtures for BASELINE configs 3 and 4, computed by the ORACLE on the CPU.

The oracle's streaming restatement (oracle/cphifi_oracle.c, SURVEY §8c mode ii: the reference's
per-observation gather/scatter of observations.hpp:174-198 fused, multiset semantics) and the
reference PCG recurrence (oracle.pcg, solvers.hpp:38-88) solve the infinite-mode subproblem
(unaligned.hpp:143-161) on the SAME seeded draws the device generates (inputs/synth_math.h; the
host generator is bit-identical to the device one, tests/test_gpu_synth.py), with K built by the
oracle's kernel functions and eig(K) / eig(V) from LAPACK (numpy).  The GPU test
(tests/test_gpu_full_pcg.py) re-runs the device solve at full size and compares against this file,
so no GPU time is spent on the oracle.

  python tests/golden/make_pcg_fixtures.py config3 [config4] [--threads T]

Writes tests/golden/<config>_pcg.npz: iterations, residual history, final relative residual,
B (the RHS sampled MTTKRP), W, A = K W (als.hpp:214), and input checksums.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from inputs import configs  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def kernel_of(cfg):
    return orc.matern32_kernel(cfg.points, cfg.ell) if cfg.kernel == "matern32" else orc.gaussian_kernel(cfg.points,
                                                                                                         cfg.ell)


def run(which, threads):
    cfg = getattr(configs, which)()
    n, r = cfg.shape[0], cfg.r
    t0 = time.perf_counter()
    idx, vals = configs.generate_host(cfg, threads=threads)
    gen_s = time.perf_counter() - t0
    kern = kernel_of(cfg)
    t0 = time.perf_counter()
    ek = orc.sym_eig(kern)
    eig_s = time.perf_counter() - t0
    factors = [np.zeros((n, r))] + cfg.factors[1:]
    t0 = time.perf_counter()
    b = orc.sampled_mttkrp_stream(cfg.shape, 0, idx, vals, factors, n, threads=threads)
    del vals
    v = orc.gram_khatri_rao(factors, 0)
    ev = orc.sym_eig(v)
    density = cfg.q / float(np.prod(np.array(cfg.shape, dtype=np.float64)))
    sub = type("Sub", (), dict(n=n, r=r, density=density, lam=cfg.lam, rho=cfg.rho, v=v))()
    m_inv = orc.build_preconditioner(sub, ek, ev)
    rhs = orc.gemm(kern, b, threads=threads).reshape(-1, order="F")   # unaligned.hpp:149-150
    nmv = [0]

    def apply_a(x):
        nmv[0] += 1
        t = time.perf_counter()
        y = orc.unaligned_matvec_stream(cfg.shape, 0, idx, factors, kern, cfg.lam, cfg.rho, x, threads=threads)
        print(f"  {which}: operator application {nmv[0]} {time.perf_counter() - t:.1f} s", file=sys.stderr, flush=True)
        return y

    rep = orc.SolveReport()
    w = orc.pcg(apply_a, lambda x: m_inv.apply(x, threads), rhs, orc.PcgConfig(cfg.tol, cfg.max_iter, True),
                rep).reshape((n, r), order="F")
    solve_s = time.perf_counter() - t0
    a = orc.gemm(kern, w, threads=threads)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), f"{which}_pcg.npz")
    np.savez_compressed(
        out, iterations=rep.iterations, relative_residual=rep.relative_residual,
        history=np.array(rep.residual_history), b=b, w=w, a=a,
        idx_checksum=np.array([int(idx[m].astype(np.int64).sum()) for m in range(idx.shape[0])]),
        q=cfg.q, threads=threads, operator_applications=nmv[0],
        seconds=np.array([gen_s, eig_s, solve_s]))
    print(f"{which}: {rep.iterations} iterations, rel {rep.relative_residual:.3e}, solve {solve_s:.0f} s "
          f"({nmv[0]} operator applications, {threads} threads) -> {out}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    args = ap.parse_args()
    for c in args.configs:
        run(c, args.threads)


if __name__ == "__main__":
    main()
