"""Pins the CPU oracle (oracle/cphifi_oracle.c + oracle/oracle.py) against every known-answer
and dense-oracle test the reference holds for this path, on the SAME seeded
instances the reference tests build (tests/refinst.py reproduces its RNG stack).

Each test names the reference test it ports (proj/tests/<file>:<lines>) and keeps its tolerance.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import refinst as ri


@pytest.fixture(scope="module", autouse=True)
def _built(built_lib):
    return built_lib


def _cp():
    """The seeded generators (inputs/): the oracle tests never load the product library."""
    import inputs
    return inputs


# ---- kernel.hpp / test_kernel.cpp --------------------------------------------------------
def test_gaussian_kernel_known_answers():
    # test_kernel.cpp:11-26
    assert np.linalg.norm(orc.gaussian_kernel([2.0, 2.0, 2.0], 1.0) - np.ones((3, 3))) < 1e-15
    assert np.linalg.norm(orc.gaussian_kernel([0.0, 1.0, 2.0], 1e6) - np.ones((3, 3))) < 1e-10
    k = orc.gaussian_kernel([0.0, 1.0], 1.0)
    assert k[0, 0] == 1.0
    assert abs(k[0, 1] - np.exp(-0.5)) < 1e-15
    assert k[0, 1] == k[1, 0]
    # test_kernel.cpp:28-31
    for s in (0.0, -1.0):
        with pytest.raises(orc.InvalidArgument):
            orc.gaussian_kernel([0.0, 1.0], s)


def test_gaussian_kernel_psd_and_grid_invariants():
    # test_kernel.cpp:33-44 and :82-89
    g = _cp().Mt19937_64(1)
    for trial in range(3):
        n = 50 + 75 * trial
        pts = g.uniform_real(0.0, 50.0, n)
        k = orc.gaussian_kernel(pts, 1.5)
        assert np.linalg.eigvalsh(k).min() > -1e-10
    k = orc.gaussian_kernel(ri.grid_points(10), 2.0)
    assert np.linalg.norm(k - k.T) < 1e-15
    assert np.linalg.norm(np.diag(k) - 1.0) < 1e-15
    e = orc.sym_eig(k)
    assert np.linalg.norm(e.u @ np.diag(e.d) @ e.u.T - k) < 1e-10 * np.linalg.norm(k)


def test_sym_eig_contract():
    # test_kernel.cpp:46-80
    e = orc.sym_eig(np.eye(4))
    assert np.linalg.norm(e.d - 1.0) < 1e-12
    e = orc.sym_eig(np.diag([3.0, 1.0]))
    assert sorted(e.d.tolist()) == [1.0, 3.0]
    g = _cp().Mt19937_64(2)
    k = ri.random_spd(g, 8)
    e = orc.sym_eig(k)
    assert np.linalg.norm(e.u @ np.diag(e.d) @ e.u.T - k) < 1e-10 * np.linalg.norm(k)
    assert np.linalg.norm(e.u.T @ e.u - np.eye(8)) < 1e-10
    assert e.d.min() >= 0.0
    with pytest.raises(orc.InvalidArgument):
        orc.sym_eig(np.array([[1.0, 2.0], [3.0, 4.0]]))


def test_matern32_definition():
    k = orc.matern32_kernel([0.0, 0.1, 0.35], 0.05)
    a = np.sqrt(3.0) * 0.25 / 0.05
    assert abs(k[2, 1] - (1 + a) * np.exp(-a)) < 1e-15
    assert np.all(np.diag(k) == 1.0) and np.array_equal(k, k.T)


# ---- observations.hpp / test_observations.cpp ----------------------------------------
def test_sampled_mttkrp_hand_expansion():
    # test_observations.cpp:180-190: out(1,0) = 7, out(1,1) = 10
    zhat = np.array([[1.0, 2.0], [3.0, 4.0]])
    out = orc.sampled_mttkrp(3, zhat, np.array([1, 1]), np.array([1.0, 2.0]))
    assert np.linalg.norm(out[0]) == 0.0 and np.linalg.norm(out[2]) == 0.0
    assert out[1, 0] == 1.0 + 2.0 * 3.0
    assert out[1, 1] == 2.0 + 2.0 * 4.0


def test_sampled_mttkrp_aligned_equals_dense():
    # test_observations.cpp:160-169 (all three modes)
    g = _cp().Mt19937_64(10)
    shape = [3, 4, 2]
    flat = ri.random_tensor(shape, g)
    factors = ri.random_model(shape, 2, g)
    idx, vals = ri.full_obs(shape, flat)
    t = flat.reshape(shape, order="F")
    for k in range(3):
        zhat = orc.build_zhat(shape, k, idx, factors)
        got = orc.sampled_mttkrp(shape[k], zhat, idx[k], vals)
        assert np.linalg.norm(got - orc.mttkrp(t, factors, k)) < 1e-12


def test_gather_rows_dense_selection_oracle():
    # test_observations.cpp:204-219
    g = _cp().Mt19937_64(13)
    shape = [3, 3, 3]
    flat = ri.random_tensor(shape, g)
    idx, _ = ri.sample(shape, flat, 8, 4)
    factors = ri.random_model(shape, 2, g)
    z = orc.khatri_rao_excluding(shape, factors, 0)
    xhat = ri.random_matrix(g, 3, 2)
    # dense S (mode-0 vec ordering) times (Z kron I_3) vec(Xhat)
    cols = idx[1].astype(np.int64) + 3 * idx[2].astype(np.int64)
    s = np.zeros((8, 27))
    s[np.arange(8), idx[0] + 3 * cols] = 1.0
    expect = s @ np.kron(z, np.eye(3)) @ xhat.reshape(-1, order="F")
    got = orc.gather_rows(xhat, orc.build_zhat(shape, 0, idx, factors), idx[0])
    assert np.abs(got - expect).max() < 1e-12


def test_zhat_matches_khatri_rao_rows():
    # test_observations.cpp:93-106: aligned Zhat rows = Z rows at the unfolding column
    g = _cp().Mt19937_64(7)
    shape = [2, 3, 4]
    flat = ri.random_tensor(shape, g)
    factors = ri.random_model(shape, 3, g)
    idx, _ = ri.full_obs(shape, flat)
    for k in range(3):
        z = orc.khatri_rao_excluding(shape, factors, k)
        zh = orc.build_zhat(shape, k, idx, factors)
        others = [m for m in range(3) if m != k]
        col = idx[others[0]].astype(np.int64) + shape[others[0]] * idx[others[1]].astype(np.int64)
        assert np.linalg.norm(zh - z[col]) < 1e-15


# ---- tensor.hpp / test_tensor_ops.cpp -------------------------------------------------
def test_mttkrp_and_gram_dense():
    # test_tensor_ops.cpp:196-227, :263-280 (shape sweep up to 5^4, r <= 4)
    g = _cp().Mt19937_64(21)
    for shape in ([3, 4, 2], [5, 5, 5, 5], [2, 3], [4, 2, 3, 2]):
        for r in (1, 3, 4):
            flat = ri.random_tensor(shape, g)
            factors = ri.random_model(shape, r, g)
            t = flat.reshape(shape, order="F")
            for k in range(len(shape)):
                # dense oracle: explicit unfolding times explicit Khatri-Rao via numpy
                others = [m for m in range(len(shape)) if m != k]
                unf = np.moveaxis(t, k, 0).reshape(shape[k], -1, order="F")
                z = np.ones((1, r))
                for m in others:  # lower modes fastest
                    z = (factors[m][:, None, :] * z[None, :, :]).reshape(-1, r)
                assert np.linalg.norm(orc.mttkrp(t, factors, k) - unf @ z) < 1e-12 * max(1, np.linalg.norm(unf @ z))
                v = np.ones((r, r))
                for m in others:
                    v *= factors[m].T @ factors[m]
                assert np.linalg.norm(orc.gram_khatri_rao(factors, k) - v) < 1e-12 * max(1, np.linalg.norm(v))


# ---- unaligned.hpp / test_unaligned_solvers.cpp + acceptance C2, C3 ---------------------
def test_matvec_empty_observations():
    # test_unaligned_solvers.cpp:131-143
    kern = orc.gaussian_kernel(ri.grid_points(3), 1.0)
    sub = orc.make_unaligned_subproblem([3, 3], np.zeros((2, 0), np.int32), np.zeros(0),
                                        [np.ones((3, 2)), np.ones((3, 2))], 0, kern, 0.5, 0.25)
    x = ri.random_matrix(_cp().Mt19937_64(4), 6, 1).reshape(-1)
    expect = 0.5 * (kern @ x.reshape((3, 2), order="F")).reshape(-1, order="F") + 0.25 * x
    assert np.linalg.norm(orc.unaligned_matvec(sub, x) - expect) < 1e-12


def test_matvec_aligned_identity_kernel_reduction():
    # test_unaligned_solvers.cpp:145-159
    g = _cp().Mt19937_64(5)
    shape = [3, 3, 3]
    flat = ri.random_tensor(shape, g)
    idx, vals = ri.full_obs(shape, flat)
    factors = ri.random_model(shape, 2, g)
    kern = orc.gaussian_kernel(ri.identity_points(3), 1.0)
    sub = orc.make_unaligned_subproblem(shape, idx, vals, factors, 0, kern, 0.3, 0.1)
    x = ri.random_matrix(g, 6, 1).reshape(-1)
    xv = (x.reshape((3, 2), order="F") @ sub.v).reshape(-1, order="F")
    assert np.linalg.norm(orc.unaligned_matvec(sub, x) - (xv + 0.3 * x + 0.1 * x)) < 1e-10


def test_matvec_dense_oracle_sweep_50_seeds():
    # test_unaligned_solvers.cpp:171-186 (exact same 50 instances)
    cp = _cp()
    for seed in range(50):
        g = cp.Mt19937_64(seed * 31 + 1)
        n = int(g.uniform_int(3, 10)[0])
        r = int(g.uniform_int(1, 4)[0])
        shape = [n, 5, 4]
        q = min(int(g.uniform_int(1, 60)[0]), n * 5 * 4)
        inst = ri.Inst(shape, r, q, 0, 1.5, 0.1, 1e-6, seed)
        dense = ri.dense_sym_operator(inst.sub)
        x = ri.random_matrix(g, n * r, 1).reshape(-1)
        expect = dense @ x
        denom = max(np.linalg.norm(expect), 1e-12)
        assert np.linalg.norm(orc.unaligned_matvec(inst.sub, x) - expect) / denom < 1e-10, seed


def test_acceptance_c2_matvec_oracle():
    # acceptance_test.cpp:149-172 (rng 202, 50 instances)
    cp = _cp()
    g = cp.Mt19937_64(202)
    worst = 0.0
    for trial in range(50):
        n = 3 + int(g() % 8)
        r = 1 + int(g() % 4)
        total = n * n * n
        q = 1 + int(g() % min(60, total))
        inst = ri.Inst([n, n, n], r, q, 0, 1.0 + 0.1 * (trial % 5), 0.1, 1e-6, None, acceptance_rng=g)
        dense = ri.dense_sym_operator(inst.sub)
        x = ri.random_matrix(g, n * r, 1).reshape(-1)
        y_ref = dense @ x
        worst = max(worst, np.linalg.norm(orc.unaligned_matvec(inst.sub, x) - y_ref) / np.linalg.norm(y_ref))
    assert worst <= 1e-10


def test_preconditioner_known_answers():
    # test_unaligned_solvers.cpp:188-199: V = I, K = I, gamma = 1 -> x / (1 + 0.3 + 0.2)
    g = _cp().Mt19937_64(8)
    flat = ri.random_tensor([3, 3], g)
    idx, vals = ri.full_obs([3, 3], flat)
    f = np.eye(3)[:, :2]
    kern = orc.gaussian_kernel(ri.identity_points(3), 1.0)
    sub = orc.make_unaligned_subproblem([3, 3], idx, vals, [f, f], 0, kern, 0.3, 0.2)
    m = orc.build_preconditioner(sub, orc.sym_eig(kern))
    x = ri.random_matrix(g, 6, 1).reshape(-1)
    assert np.linalg.norm(m.apply(x) - x / (1.0 + 0.3 + 0.2)) < 1e-12


def test_preconditioner_dense_oracle():
    # test_unaligned_solvers.cpp:201-217
    g = _cp().Mt19937_64(9)
    for trial in range(20):
        inst = ri.Inst([8, 4, 3], 3, 30, 0, 1.5, 0.1, 1e-6, trial + 100)
        dense_inv = np.linalg.inv(ri.dense_preconditioner(inst.sub))
        m = orc.build_preconditioner(inst.sub, orc.sym_eig(inst.kernel))
        x = ri.random_matrix(g, 24, 1).reshape(-1)
        expect = dense_inv @ x
        assert np.linalg.norm(m.apply(x) - expect) / np.linalg.norm(expect) < 1e-8


def test_acceptance_c3_preconditioner_and_full_density():
    # acceptance_test.cpp:174-218
    cp = _cp()
    g = cp.Mt19937_64(303)
    worst = 0.0
    for _ in range(20):
        n = 4 + int(g() % 8)
        r = 1 + int(g() % 4)
        q = 1 + int(g() % min(120, n ** 3))
        inst = ri.Inst([n, n, n], r, q, 0, 1.2, 0.1, 1e-4, None, acceptance_rng=g)
        m = ri.dense_preconditioner(inst.sub)
        pre = orc.build_preconditioner(inst.sub, orc.sym_eig(inst.kernel))
        x = ri.random_matrix(g, n * r, 1).reshape(-1)
        y_ref = np.linalg.solve(m, x)
        worst = max(worst, np.linalg.norm(pre.apply(x) - y_ref) / np.linalg.norm(y_ref))
    assert worst <= 1e-8
    worst_iters = 0
    for lam in (0.05, 0.5):
        for rho in (1e-6, 1e-2):
            flat = ri.random_tensor([6, 5, 5], g)
            idx, vals = ri.full_obs([6, 5, 5], flat)
            factors = ri.random_model([6, 5, 5], 3, g)
            kern = orc.gaussian_kernel(ri.grid_points(6), 1.5)
            sub = orc.make_unaligned_subproblem([6, 5, 5], idx, vals, factors, 0, kern, lam, rho)
            rep = orc.SolveReport()
            orc.solve_unaligned_pcg(sub, orc.PcgConfig(1e-10, 75), orc.sym_eig(kern), report=rep)
            worst_iters = max(worst_iters, rep.iterations)
    assert worst_iters <= 2


def test_pcg_matches_dense_cholesky_and_row_order():
    # test_unaligned_solvers.cpp:248-257 and :309-329
    inst = ri.Inst([20, 6, 5], 4, 400, 0, 0.8, 0.1, 1e-6, 11)
    sysm = ri.dense_sym_operator(inst.sub)
    rhs = (inst.kernel @ inst.sub.b).reshape(-1, order="F")
    w_ref = np.linalg.solve(sysm, rhs)
    w = orc.solve_unaligned_pcg(inst.sub, orc.PcgConfig(1e-10, 200), orc.sym_eig(inst.kernel))
    assert ri.rel(w.reshape(-1, order="F"), w_ref) < 1e-5
    inst2 = ri.Inst([6, 5, 4], 2, 40, 0, 1.0, 0.1, 1e-6, 15)
    ek = orc.sym_eig(inst2.kernel)
    w1 = orc.solve_unaligned_pcg(inst2.sub, orc.PcgConfig(1e-10, 200), ek)
    perm = np.random.default_rng(99).permutation(inst2.sub.q)
    sub2 = orc.make_unaligned_subproblem(inst2.shape, inst2.idx[:, perm], inst2.vals[perm], inst2.factors, 0,
                                         inst2.kernel, 0.1, 1e-6)
    w2 = orc.solve_unaligned_pcg(sub2, orc.PcgConfig(1e-10, 200), ek)
    assert ri.rel(w2, w1) < 1e-8


def test_pcg_zero_rhs_and_exact_full_density():
    # test_unaligned_solvers.cpp:237-246 and :219-235
    kern = orc.gaussian_kernel(ri.grid_points(3), 1.0)
    sub = orc.make_unaligned_subproblem([3, 3], np.array([[0], [0]]), np.array([0.0]),
                                        [np.ones((3, 2)), np.ones((3, 2))], 0, kern, 0.5, 1e-6)
    rep = orc.SolveReport()
    w = orc.solve_unaligned_pcg(sub, orc.PcgConfig(), orc.sym_eig(kern), report=rep)
    assert np.linalg.norm(w) < 1e-14 and rep.iterations <= 1
    g = _cp().Mt19937_64(10)
    flat = ri.random_tensor([5, 4, 3], g)
    idx, vals = ri.full_obs([5, 4, 3], flat)
    factors = ri.random_model([5, 4, 3], 2, g)
    for lam in (0.01, 0.5):
        for rho in (1e-6, 0.1):
            kern = orc.gaussian_kernel(ri.grid_points(5), 1.5)
            sub = orc.make_unaligned_subproblem([5, 4, 3], idx, vals, factors, 0, kern, lam, rho)
            rep = orc.SolveReport()
            orc.solve_unaligned_pcg(sub, orc.PcgConfig(1e-8, 75), orc.sym_eig(kern), report=rep)
            assert rep.iterations <= 2


# ---- solvers.hpp / test_linear_solvers.cpp ------------------------------------------------
def test_pcg_contract():
    cp = _cp()
    ident = lambda v: v.copy()
    # :20-29 identity -> exactly one iteration
    b = ri.random_matrix(cp.Mt19937_64(1), 10, 1).reshape(-1)
    rep = orc.SolveReport()
    x = orc.pcg(ident, ident, b, orc.PcgConfig(), rep)
    assert np.linalg.norm(x - b) < 1e-12 and rep.iterations == 1 and rep.converged
    # :31-44 exact preconditioner -> <= 1 iteration
    dvec = np.arange(1, 11, dtype=np.float64)
    b = ri.random_matrix(cp.Mt19937_64(2), 10, 1).reshape(-1)
    rep = orc.SolveReport()
    x = orc.pcg(lambda v: dvec * v, lambda v: v / dvec, b, orc.PcgConfig(1e-10, 75), rep)
    assert rep.iterations <= 1 and np.linalg.norm(dvec * x - b) / np.linalg.norm(b) < 1e-10
    # :61-68 zero rhs -> 0 iterations, converged
    rep = orc.SolveReport()
    x = orc.pcg(ident, ident, np.zeros(5), orc.PcgConfig(), rep)
    assert np.linalg.norm(x) == 0.0 and rep.converged and rep.iterations == 0
    # :70-75 indefinite throws runtime_error
    with pytest.raises(orc.RuntimeFailure):
        orc.pcg(lambda v: -v, ident, np.ones(4), orc.PcgConfig())
    # :46-59 matches dense solve within tol * kappa
    g = cp.Mt19937_64(3)
    a = ri.random_spd(g, 50, 1.0)
    b = ri.random_matrix(g, 50, 1).reshape(-1)
    rep = orc.SolveReport()
    x = orc.pcg(lambda v: a @ v, ident, b, orc.PcgConfig(1e-10, 200), rep)
    ev = np.linalg.eigvalsh(a)
    assert ri.rel(x, np.linalg.solve(a, b)) < 1e-10 * ev.max() / ev.min() and rep.converged
    # :77-92 A-norm error monotone
    g = cp.Mt19937_64(4)
    a = ri.random_spd(g, 30, 1.0)
    xt = ri.random_matrix(g, 30, 1).reshape(-1)
    b = a @ xt
    prev = np.inf
    for iters in range(1, 11):
        x = orc.pcg(lambda v: a @ v, ident, b, orc.PcgConfig(1e-14, iters))
        e = x - xt
        an = np.sqrt(e @ (a @ e))
        assert an <= prev * (1 + 1e-12)
        prev = an


# ---- aligned.hpp / test_aligned_solvers.cpp + acceptance C1 --------------------------------
def _direct_aligned(b, v, kern, lam):
    sysm = np.kron(v, kern) + lam * np.eye(b.size)
    return np.linalg.solve(sysm, b.reshape(-1, order="F")).reshape(b.shape, order="F")


def test_decoupled_known_answers():
    cp = _cp()
    # test_aligned_solvers.cpp:73-81: identity system -> W = B / 2
    g = cp.Mt19937_64(4)
    b = ri.random_matrix(g, 4, 2)
    kern = orc.gaussian_kernel(ri.identity_points(4), 1.0)
    w = orc.solve_aligned_decoupled(b, orc.sym_eig(kern), orc.sym_eig(np.eye(2)), 1.0)
    assert np.linalg.norm(w - 0.5 * b) < 1e-10
    # :83-96: lambda = 0, diagonal K and V -> W(i,j) = B(i,j) / V(j,j)
    g = cp.Mt19937_64(5)
    b = ri.random_matrix(g, 3, 2)
    v = np.diag([2.0, 5.0])
    kern = orc.gaussian_kernel(ri.identity_points(3), 1.0)
    w = orc.solve_aligned_decoupled(b, orc.sym_eig(kern), orc.sym_eig(v), 0.0)
    assert np.abs(w - b / np.diag(v)[None, :]).max() < 1e-10
    # zero eigenvalue pair with lambda = 0 throws runtime_error (aligned.hpp:48-50)
    with pytest.raises(orc.RuntimeFailure):
        orc.solve_aligned_decoupled(b, orc.sym_eig(kern), orc.sym_eig(np.zeros((2, 2))), 0.0)


def test_acceptance_c1_decoupled_vs_direct():
    # acceptance_test.cpp:117-147 (decoupled part) and test_aligned_solvers.cpp:98-104
    g = _cp().Mt19937_64(101)
    grid = [(n, r, lam) for n in (10, 20, 40) for r in (2, 5, 8) for lam in (0.1, 1.0)]
    grid += [(30, 6, 0.1), (25, 4, 1.0)]
    worst = 0.0
    for n, r, lam in grid:
        b = ri.random_matrix(g, n, r)
        v = ri.random_spd(g, r)
        kern = orc.gaussian_kernel(ri.grid_points(n), 2.0)
        wd = _direct_aligned(b, v, kern, lam)
        wdec = orc.solve_aligned_decoupled(b, orc.sym_eig(kern), orc.sym_eig(v), lam)
        worst = max(worst, ri.rel(wdec, wd))
    assert worst <= 1e-8
