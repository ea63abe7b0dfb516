"""The aligned subproblem's comparison solvers: aligned_matvec, solve_aligned_pcg
and solve_aligned_direct (aligned.hpp:28-100).

CPU tests pin the oracle restatement (oracle/oracle.py) against the reference's own known-answer
tests, on the same seeded instances (tests/refinst.py reproduces its RNG stack); GPU tests run the
device implementations (k_aligned.cu through the C-ABI) on those instances and against the oracle
on larger ones.  Each test names the reference test it ports and keeps its tolerance.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import refinst as ri


@pytest.fixture(scope="module", autouse=True)
def _built(built_lib):
    return built_lib


def _cp():
    import paper_2603_25691_b200 as cp
    return cp


def _grid_kernel(n, sigma):  # RkhsMode::regular_grid (kernel.hpp:64-68): points 1..n
    return orc.gaussian_kernel(ri.grid_points(n), sigma)


def _random_problem(n, r, sigma, lam, seed):
    """random_problem (test_aligned_solvers.cpp:26-33): B, then V = random_spd, grid mode."""
    rng = _cp().Mt19937_64(seed)
    b = ri.random_matrix(rng, n, r)
    v = ri.random_spd(rng, r)
    return b, v, _grid_kernel(n, sigma), lam


# ---- oracle pinned against the reference tests (CPU) ---------------------------------------
def test_oracle_direct_identity_system():
    # test_aligned_solvers.cpp:37-45: K = I, V = I, lambda = 1 -> W = B / 2
    rng = _cp().Mt19937_64(1)
    b = ri.random_matrix(rng, 4, 2)
    w = orc.solve_aligned_direct(b, orc.gaussian_kernel(ri.identity_points(4), 1.0), np.eye(2), 1.0)
    assert np.linalg.norm(w - 0.5 * b) < 1e-12


def test_oracle_direct_rank_one_and_residual():
    # test_aligned_solvers.cpp:47-63
    rng = _cp().Mt19937_64(2)
    b = ri.random_matrix(rng, 6, 1)
    k = _grid_kernel(6, 1.5)
    w = orc.solve_aligned_direct(b, k, np.ones((1, 1)), 0.3)
    assert np.linalg.norm((k + 0.3 * np.eye(6)) @ w - b) < 1e-9 * np.linalg.norm(b)
    b, v, k, lam = _random_problem(12, 3, 2.0, 0.1, 3)
    w = orc.solve_aligned_direct(b, k, v, lam)
    assert orc.aligned_residual_dense(b, k, v, lam, w) < 1e-9


def test_oracle_direct_memory_guard():
    # test_aligned_solvers.cpp:65-71
    with pytest.raises(orc.InvalidArgument):
        orc.solve_aligned_direct(np.ones((100, 100)), _grid_kernel(100, 1.0), np.eye(100), 0.1)


def test_oracle_aligned_matvec():
    # test_aligned_solvers.cpp:106-124
    rng = _cp().Mt19937_64(7)
    x = ri.random_matrix(rng, 12, 1).reshape(-1)
    dk = np.ones(4)
    assert np.linalg.norm(orc.aligned_matvec(x, dk, np.eye(3), 0.0) - x) < 1e-14
    assert np.linalg.norm(orc.aligned_matvec(x, dk, np.zeros((3, 3)), 2.5) - 2.5 * x) < 1e-14
    rng = _cp().Mt19937_64(8)
    dk = np.abs(ri.random_matrix(rng, 8, 1).reshape(-1))
    v = ri.random_spd(rng, 3)
    dense = np.kron(v, np.diag(dk)) + 0.7 * np.eye(24)
    x = ri.random_matrix(rng, 24, 1).reshape(-1)
    assert np.linalg.norm(orc.aligned_matvec(x, dk, v, 0.7) - dense @ x) < 1e-12


def test_oracle_pcg_known_answers():
    # test_aligned_solvers.cpp:126-161
    rng = _cp().Mt19937_64(9)
    b = ri.random_matrix(rng, 4, 2)
    ek = orc.sym_eig(orc.gaussian_kernel(ri.identity_points(4), 1.0))
    rep = orc.SolveReport()
    w = orc.solve_aligned_pcg(b, ek, np.eye(2), 1.0, orc.PcgConfig(1e-10, 75), rep)
    assert np.linalg.norm(w - 0.5 * b) < 1e-9 and rep.iterations <= 2
    rng = _cp().Mt19937_64(10)
    b = ri.random_matrix(rng, 6, 3)
    rep = orc.SolveReport()
    orc.solve_aligned_pcg(b, orc.sym_eig(_grid_kernel(6, 1.5)), np.diag([1.0, 2.0, 3.0]), 0.2,
                          orc.PcgConfig(1e-10, 75), rep)
    assert rep.iterations <= 2
    b, v, k, lam = _random_problem(40, 8, 2.0, 0.1, 11)
    ek = orc.sym_eig(k)
    rep = orc.SolveReport()
    wp = orc.solve_aligned_pcg(b, ek, v, lam, orc.PcgConfig(1e-8, 75), rep)
    wd = orc.solve_aligned_decoupled(b, ek, orc.sym_eig(v), lam)
    assert np.linalg.norm(wp - wd) / np.linalg.norm(wd) < 1e-5 and rep.iterations <= 75


def test_oracle_decoupled_matches_direct():
    # test_aligned_solvers.cpp:98-104
    b, v, k, lam = _random_problem(30, 5, 2.0, 0.1, 6)
    wd = orc.solve_aligned_direct(b, k, v, lam)
    wdec = orc.solve_aligned_decoupled(b, orc.sym_eig(k), orc.sym_eig(v), lam)
    assert np.linalg.norm(wd - wdec) / np.linalg.norm(wd) < 1e-8


# ---- device implementations (GPU) ---------------------------------------------------------
def _mode(cp, points, sigma, lam):
    return cp.RkhsMode(points, sigma, lam)


@pytest.mark.gpu
def test_device_aligned_matvec(ctx):
    cp = _cp()
    rng = cp.Mt19937_64(8)
    dk = np.abs(ri.random_matrix(rng, 8, 1).reshape(-1))
    v = ri.random_spd(rng, 3)
    x = ri.random_matrix(rng, 24, 1).reshape(-1)
    dense = np.kron(v, np.diag(dk)) + 0.7 * np.eye(24)
    assert np.linalg.norm(cp.aligned_matvec(x, dk, v, 0.7) - dense @ x) < 1e-12
    g = np.random.default_rng(3)
    dk, v, x = g.random(300), g.normal(size=(17, 17)), g.normal(size=300 * 17)
    assert ri.rel(cp.aligned_matvec(x, dk, v, 0.3), orc.aligned_matvec(x, dk, v, 0.3)) < 1e-14
    with pytest.raises(cp.CphifiInvalidArgument):
        cp.aligned_matvec(x[:-1], dk, v, 0.3)


@pytest.mark.gpu
def test_device_direct_known_answers(ctx):
    cp = _cp()
    rng = cp.Mt19937_64(1)
    b = ri.random_matrix(rng, 4, 2)
    w = cp.solve_aligned_direct(cp.AlignedSubproblem(b, np.eye(2), _mode(cp, ri.identity_points(4), 1.0, 1.0)))
    assert np.linalg.norm(w - 0.5 * b) < 1e-12
    b, v, k, lam = _random_problem(12, 3, 2.0, 0.1, 3)
    w = cp.solve_aligned_direct(cp.AlignedSubproblem(b, v, _mode(cp, ri.grid_points(12), 2.0, lam)))
    assert orc.aligned_residual_dense(b, k, v, lam, w) < 1e-9
    assert ri.rel(w, orc.solve_aligned_direct(b, k, v, lam)) < 1e-11
    with pytest.raises(cp.CphifiInvalidArgument, match="rn exceeds memory cap"):
        cp.solve_aligned_direct(cp.AlignedSubproblem(np.ones((100, 100)), np.eye(100),
                                                     _mode(cp, ri.grid_points(100), 1.0, 0.1)))
    with pytest.raises(cp.CphifiRuntimeError, match="not positive definite"):  # lambda < -min eig
        cp.solve_aligned_direct(cp.AlignedSubproblem(b, -np.eye(3), _mode(cp, ri.grid_points(12), 2.0, 0.1)))


@pytest.mark.gpu
def test_device_pcg_known_answers(ctx):
    cp = _cp()
    rng = cp.Mt19937_64(9)
    b = ri.random_matrix(rng, 4, 2)
    rep = cp.SolveReport()
    w = cp.solve_aligned_pcg(cp.AlignedSubproblem(b, np.eye(2), _mode(cp, ri.identity_points(4), 1.0, 1.0)),
                             cp.PcgConfig(1e-10, 75), rep)
    assert np.linalg.norm(w - 0.5 * b) < 1e-9 and rep.iterations <= 2
    rng = cp.Mt19937_64(10)
    b = ri.random_matrix(rng, 6, 3)
    rep = cp.SolveReport()
    cp.solve_aligned_pcg(cp.AlignedSubproblem(b, np.diag([1.0, 2.0, 3.0]), _mode(cp, ri.grid_points(6), 1.5, 0.2)),
                         cp.PcgConfig(1e-10, 75), rep)
    assert rep.iterations <= 2
    rep = cp.SolveReport()
    zero = cp.solve_aligned_pcg(cp.AlignedSubproblem(np.zeros((6, 3)), np.eye(3), _mode(cp, ri.grid_points(6), 1.5, 0.2)),
                                cp.PcgConfig(1e-10, 75), rep)
    assert rep.iterations == 0 and rep.converged and not zero.any()  # solvers.hpp:49-53


@pytest.mark.gpu
@pytest.mark.parametrize("n,r,seed", [(40, 8, 11), (300, 12, 12)])
def test_device_pcg_vs_oracle(ctx, n, r, seed):
    """Same eig(K) on both sides: iteration counts within +-1, W to the solve tolerance,
    residual history element-wise; a warm start from the solution converges at once."""
    cp = _cp()
    b, v, k, lam = _random_problem(n, r, 2.0, 0.1, seed)
    mode = _mode(cp, ri.grid_points(n), 2.0, lam)
    ek = orc.sym_eig(k)
    mode.set_eig(ek.u, ek.d)
    cfg = cp.PcgConfig(1e-9, 200, record_history=True)
    rep, orep = cp.SolveReport(), orc.SolveReport()
    p = cp.AlignedSubproblem(b, v, mode)
    w = cp.solve_aligned_pcg(p, cfg, rep)
    wo = orc.solve_aligned_pcg(b, ek, v, lam, orc.PcgConfig(1e-9, 200, record_history=True), orep)
    assert rep.converged and abs(rep.iterations - orep.iterations) <= 1, (rep.iterations, orep.iterations)
    assert ri.rel(w, wo) < 1e-7
    m = min(len(rep.residual_history), len(orep.residual_history))
    h, ho = np.asarray(rep.residual_history[:m]), np.asarray(orep.residual_history[:m])
    assert np.all(np.abs(h - ho) <= 1e-6 * ho + 1e-14)
    wdec = cp.solve_aligned_decoupled(p, orc.sym_eig(v))
    assert ri.rel(w, wdec) < 1e-5
    rep2 = cp.SolveReport()
    cp.solve_aligned_pcg(p, cfg, rep2, warm_start=w)
    assert rep2.iterations <= 1
