"""The unaligned direct / dense baselines (unaligned.hpp:52-96, 164-174).

CPU: the oracle's restatement pinned by ports of the reference tests that hold them
(test_unaligned_solvers.cpp: BuildF.*, SolveUnalignedDirectNonsym.*, AssembleUnalignedSymDense.Examples,
UnalignedSolvers.CrossSolverAgreement) on the same seeded instances.
GPU: the device versions (systems assembled from the row Grams) against the oracle."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import refinst as ri
from inputs import Mt19937_64


def _sub(shape, idx, vals, factors, k, kern, lam, rho):
    return orc.make_unaligned_subproblem(shape, idx, vals, factors, k, kern, lam, rho)


# ---- CPU: the oracle, pinned by the reference's own tests --------------------------------------
def test_buildF_identity_kernel_gives_G():
    rng = Mt19937_64(1)
    t = ri.random_tensor([4, 4, 4], rng)
    idx, vals = ri.sample([4, 4, 4], t, 12, 2)
    m = ri.random_model([4, 4, 4], 2, rng)
    sub = _sub([4, 4, 4], idx, vals, m, 1, orc.gaussian_kernel(ri.identity_points(4), 0.1), 0.1, 1e-6)
    assert np.linalg.norm(orc.build_F(sub) - orc.build_G(sub)) < 1e-12


def test_buildF_aligned_equals_dense_kronecker():
    rng = Mt19937_64(2)
    shape = [3, 3, 2]
    t = ri.random_tensor(shape, rng)
    idx, vals = ri.full_obs(shape, t)
    m = ri.random_model(shape, 2, rng)
    kern = orc.gaussian_kernel(ri.grid_points(3), 1.0)
    sub = _sub(shape, idx, vals, m, 0, kern, 0.1, 1e-6)
    z = orc.khatri_rao_excluding(shape, m, 0)  # rows: i1 + n1 i2 (tensor.hpp:158-165)
    zk = np.kron(z, kern)                      # row (z_row, i0) = z_row n + i0
    sel = (idx[1] + 3 * idx[2]) * 3 + idx[0]   # S' picks observation l's row
    assert np.linalg.norm(orc.build_F(sub) - zk[sel]) < 1e-12
    assert np.linalg.norm(orc.build_G(sub) - np.kron(z, np.eye(3))[sel]) < 1e-12


def test_buildF_single_observation_row():
    kern = orc.gaussian_kernel(ri.grid_points(2), 1.0)
    sub = _sub([2, 2], np.array([[1], [0]]), np.array([2.0]), [np.ones((2, 1)), np.ones((2, 1))], 0, kern, 0.1, 1e-6)
    f = orc.build_F(sub)
    assert f.shape[0] == 1 and np.linalg.norm(f[0] - kern[1]) < 1e-12


def test_direct_nonsym_aligned_reduces_to_aligned_direct():
    rng = Mt19937_64(3)
    shape = [4, 3, 3]
    t = ri.random_tensor(shape, rng)
    idx, vals = ri.full_obs(shape, t)
    m = ri.random_model(shape, 2, rng)
    kern = orc.gaussian_kernel(ri.grid_points(4), 1.5)
    sub = _sub(shape, idx, vals, m, 0, kern, 0.2, 1e-6)
    w = orc.solve_unaligned_direct_nonsym(sub)
    b = orc.mttkrp(t.reshape(shape, order="F"), m, 0)
    wa = orc.solve_aligned_direct(b, kern, orc.gram_khatri_rao(m, 0), 0.2)
    assert np.linalg.norm(w - wa) / np.linalg.norm(wa) < 1e-8


def test_direct_nonsym_empty_and_residual_and_cap():
    kern = orc.gaussian_kernel(ri.grid_points(3), 1.0)
    sub0 = _sub([3, 3], np.zeros((2, 0), np.int32), np.zeros(0), [np.ones((3, 2)), np.ones((3, 2))], 0, kern, 0.5,
                1e-6)
    assert np.linalg.norm(orc.solve_unaligned_direct_nonsym(sub0)) < 1e-14
    inst = ri.Inst([5, 5, 5], 2, 40, 0, 1.0, 0.1, 1e-6, 42)
    rep = orc.SolveReport()
    w = orc.solve_unaligned_direct_nonsym(inst.sub, rep)
    sys_ = orc.build_G(inst.sub).T @ orc.build_F(inst.sub)
    sys_[np.diag_indices_from(sys_)] += 0.1
    bv = inst.sub.b.reshape(-1, order="F")
    assert np.linalg.norm(sys_ @ w.reshape(-1, order="F") - bv) / np.linalg.norm(bv) < 1e-9
    assert rep.iterations == 1 and rep.relative_residual < 1e-9
    with pytest.raises(orc.InvalidArgument, match="rn exceeds memory cap"):
        orc.solve_unaligned_direct_nonsym(inst.sub, dense_cap=9)


def test_assemble_sym_dense_examples():
    kern = orc.gaussian_kernel(ri.grid_points(3), 1.0)
    p0 = _sub([3, 3], np.zeros((2, 0), np.int32), np.zeros(0), [np.ones((3, 2)), np.ones((3, 2))], 0, kern, 0.4, 0.2)
    sys0, rhs0 = orc.assemble_unaligned_sym_dense(p0)
    expect0 = 0.4 * np.kron(np.eye(2), kern) + 0.2 * np.eye(6)
    assert np.linalg.norm(sys0 - expect0) < 1e-12 and np.linalg.norm(rhs0) < 1e-14
    rng = Mt19937_64(13)
    shape = [4, 3, 3]
    t = ri.random_tensor(shape, rng)
    idx, vals = ri.full_obs(shape, t)
    m2 = ri.random_model(shape, 2, rng)
    k4 = orc.gaussian_kernel(ri.grid_points(4), 1.5)
    p = _sub(shape, idx, vals, m2, 0, k4, 0.3, 0.1)
    sys_, rhs = orc.assemble_unaligned_sym_dense(p)
    expect = np.kron(p.v, k4 @ k4) + 0.3 * np.kron(np.eye(2), k4) + 0.1 * np.eye(8)
    assert np.linalg.norm(sys_ - expect) / np.linalg.norm(expect) < 1e-10
    assert np.linalg.norm(sys_ - sys_.T) < 1e-12


def test_cross_solver_agreement():
    inst = ri.Inst([10, 6, 5], 3, 150, 0, 0.5, 0.1, 1e-6, 14)
    w_ns = orc.solve_unaligned_direct_nonsym(inst.sub)
    ek = orc.sym_eig(inst.kernel)
    w_pcg = orc.solve_unaligned_pcg(inst.sub, orc.PcgConfig(1e-10, 300), ek)
    assert np.linalg.norm(w_pcg - w_ns) / np.linalg.norm(w_ns) < max(1e-4, 10.0 * 1e-6 / 0.1)


# ---- GPU: the device versions against the oracle ---------------------------------------------
def _device(inst):
    import paper_2603_25691_b200 as cp
    mode = cp.RkhsMode(inst.points, inst.sigma, inst.lam, kernel_matrix=inst.kernel)
    obs = cp.ObservationSet(inst.shape, inst.idx, inst.vals)
    return cp, cp.make_unaligned_subproblem(obs, cp.KruskalModel(inst.factors), inst.k, mode, inst.rho)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(10))
def test_device_direct_nonsym_and_sym_dense(seed):
    g = Mt19937_64(seed * 7 + 3)
    shape = [int(g.uniform_int(3, 12)[0]), int(g.uniform_int(2, 6)[0]), int(g.uniform_int(2, 6)[0])]
    r = int(g.uniform_int(1, 4)[0])
    q = int(g.uniform_int(1, int(np.prod(shape)))[0])
    inst = ri.Inst(shape, r, q, 0, 0.8, 0.1, 1e-6, 100 + seed)
    cp, p = _device(inst)
    rep = cp.SolveReport()
    w = cp.solve_unaligned_direct_nonsym(p, rep)
    wo = orc.solve_unaligned_direct_nonsym(inst.sub)
    assert np.linalg.norm(w - wo) / max(np.linalg.norm(wo), 1e-300) < 1e-9
    assert rep.iterations == 1 and rep.relative_residual < 1e-9
    sys_, rhs = cp.assemble_unaligned_sym_dense(p)
    so, ro = orc.assemble_unaligned_sym_dense(inst.sub)
    assert np.linalg.norm(sys_ - so) / np.linalg.norm(so) < 1e-12
    assert np.linalg.norm(rhs - ro) / max(np.linalg.norm(ro), 1e-300) < 1e-12


@pytest.mark.gpu
def test_device_direct_contract():
    import paper_2603_25691_b200 as cp
    inst = ri.Inst([40, 6, 5], 4, 300, 0, 0.8, 0.1, 1e-6, 5)
    cp, p = _device(inst)
    with pytest.raises(cp.CphifiInvalidArgument, match="rn exceeds memory cap"):
        cp.solve_unaligned_direct_nonsym(p, dense_cap=100)
    with pytest.raises(cp.CphifiInvalidArgument, match="assemble_unaligned_sym_dense: rn exceeds memory cap"):
        cp.assemble_unaligned_sym_dense(p, dense_cap=100)
    # empty observations: W = 0 (test_unaligned_solvers.cpp:112-119)
    kern = orc.gaussian_kernel(ri.grid_points(3), 1.0)
    mode = cp.RkhsMode(ri.grid_points(3), 1.0, 0.5, kernel_matrix=kern)
    obs = cp.ObservationSet([3, 3], np.zeros((2, 0), np.int32), np.zeros(0))
    p0 = cp.make_unaligned_subproblem(obs, cp.KruskalModel([np.ones((3, 2)), np.ones((3, 2))]), 0, mode, 1e-6)
    assert np.linalg.norm(cp.solve_unaligned_direct_nonsym(p0)) < 1e-14
    # a singular system: lambda = 0 and no observations
    mode_z = cp.RkhsMode(ri.grid_points(3), 1.0, 0.0, kernel_matrix=kern)
    pz = cp.make_unaligned_subproblem(obs, cp.KruskalModel([np.ones((3, 2)), np.ones((3, 2))]), 0, mode_z, 1e-6)
    with pytest.raises(cp.CphifiRuntimeError, match="lu_solve: matrix is singular"):
        cp.solve_unaligned_direct_nonsym(pz)
    with pytest.raises(orc.RuntimeFailure, match="lu_solve: matrix is singular"):
        orc.solve_unaligned_direct_nonsym(orc.make_unaligned_subproblem(
            [3, 3], np.zeros((2, 0), np.int32), np.zeros(0), [np.ones((3, 2)), np.ones((3, 2))], 0, kern, 0.0, 1e-6))
