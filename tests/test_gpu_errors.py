"""The reference's runtime-error contract provoked on the device, next to the oracle on the same
instance (SURVEY §8b errors):
  * "pcg: non-finite value encountered"            (solvers.hpp:65-66): p'Ap is not finite;
  * "pcg: operator not positive definite (p'Ap <= 0)" (solvers.hpp:67-68): an indefinite kernel K;
  * "build_preconditioner: nonpositive denominator" (unaligned.hpp:130-131): rho = 0 with a clamped
    eigenvalue mu_i = 0 of K.
Each at a small n (the fused single-launch operator, device-resident PCG graph) and a large n (GEMMs
around the streaming pass)."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _instance(n, seed=3):
    g = np.random.default_rng(seed)
    shape = [n, 9, 7]
    r = 4
    q = 6 * n
    lin = g.choice(n * 9 * 7, size=q, replace=False)
    idx = np.stack([lin % n, (lin // n) % 9, lin // (n * 9)]).astype(np.int32)
    vals = g.normal(size=q)
    factors = [np.zeros((n, r))] + [g.normal(size=(s, r)) for s in shape[1:]]
    return shape, r, idx, vals, factors


def _device(shape, r, idx, vals, factors, kern, lam, rho):
    import paper_2603_25691_b200 as cp
    mode = cp.RkhsMode(np.arange(shape[0], dtype=float), 1.0, lam, kernel_matrix=kern)
    obs = cp.ObservationSet(shape, idx, vals)
    return cp, cp.make_unaligned_subproblem(obs, cp.KruskalModel(factors), 0, mode, rho)


def _oracle(shape, idx, vals, factors, kern, lam, rho):
    return orc.make_unaligned_subproblem(shape, idx, vals, factors, 0, kern, lam, rho)


@pytest.mark.parametrize("n", [40, 600])
def test_nonfinite_pap(n):
    shape, r, idx, vals, factors = _instance(n)
    pts = np.sort(np.random.default_rng(1).uniform(size=n))
    kern = orc.gaussian_kernel(pts, 0.1)
    cp, p = _device(shape, r, idx, vals, factors, kern, 1e-3, 1e-6)
    x0 = np.full((n, r), 1e300)  # A x0 overflows: r0 = b - A x0 is infinite, p'Ap is NaN
    with pytest.raises(cp.CphifiRuntimeError, match="pcg: non-finite value encountered"):
        cp.solve_unaligned_pcg(p, cp.PcgConfig(1e-8, 50), warm_start=x0)
    sub = _oracle(shape, idx, vals, factors, kern, 1e-3, 1e-6)
    with pytest.raises(orc.RuntimeFailure, match="pcg: non-finite value encountered"):
        orc.solve_unaligned_pcg(sub, orc.PcgConfig(1e-8, 50), orc.sym_eig(kern), warm_start=x0)


@pytest.mark.parametrize("n", [40, 600])
def test_indefinite_operator(n):
    shape, r, idx, vals, factors = _instance(n)
    kern = -np.eye(n)  # lambda (I kron K) = -100 I dominates: the operator is negative definite
    cp, p = _device(shape, r, idx, vals, factors, kern, 100.0, 1e-6)
    with pytest.raises(cp.CphifiRuntimeError, match=r"pcg: operator not positive definite \(p'Ap <= 0\)"):
        cp.solve_unaligned_pcg(p, cp.PcgConfig(1e-8, 50))
    sub = _oracle(shape, idx, vals, factors, kern, 100.0, 1e-6)
    with pytest.raises(orc.RuntimeFailure, match=r"pcg: operator not positive definite"):
        orc.solve_unaligned_pcg(sub, orc.PcgConfig(1e-8, 50), orc.sym_eig(kern))


@pytest.mark.parametrize("n", [40, 600])
def test_nonpositive_preconditioner_denominator(n):
    shape, r, idx, vals, factors = _instance(n)
    kern = np.zeros((n, n))  # every eigenvalue clamps to 0: with rho = 0 every denominator is 0
    cp, p = _device(shape, r, idx, vals, factors, kern, 1e-3, 0.0)
    with pytest.raises(cp.CphifiRuntimeError, match="build_preconditioner: nonpositive denominator"):
        cp.build_preconditioner(p)
    sub = _oracle(shape, idx, vals, factors, kern, 1e-3, 0.0)
    with pytest.raises(orc.RuntimeFailure, match="build_preconditioner: nonpositive denominator"):
        orc.build_preconditioner(sub, orc.sym_eig(kern))
    # the solve itself rejects rho <= 0 first (unaligned.hpp:146-147)
    with pytest.raises(cp.CphifiInvalidArgument, match="rho must be positive"):
        cp.solve_unaligned_pcg(p, cp.PcgConfig(1e-8, 50))
