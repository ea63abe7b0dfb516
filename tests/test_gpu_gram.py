"""Row-Gram form of the unaligned operator (k_gram.cu) against the CPU oracle.

Yhat(i,:) = G_i Xhat(i,:) with G_i = sum_{l in row i} z_l z_l' is an exact identity of the
reference's gather/scatter (observations.hpp:174-198); only the fp64 association changes, so the
bar is 1e-12 relative like the streaming operator, PCG iterations within +-1 of the oracle and
the final residual <= tol.
"""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import refinst as ri

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cp(ctx):
    import paper_2603_25691_b200 as cp
    return cp


@pytest.mark.parametrize("shape,r,q", [([57, 9, 8], 3, 2000), ([33, 7, 6, 5], 8, 3000), ([20, 30], 17, 500),
                                       ([64, 10, 11], 32, 5000), ([31, 12, 9], 64, 3000), ([12, 40, 40], 10, 1)])
def test_gram_matvec_vs_oracle(cp, shape, r, q):
    inst = ri.Inst(shape, r, q, 0, 0.7, 0.1, 1e-6, 99 + r)
    mode = cp.RkhsMode(inst.points, inst.sigma, inst.lam)
    inst.sub.kernel = mode.kernel()
    p = cp.make_unaligned_subproblem(cp.ObservationSet(inst.shape, inst.idx, inst.vals),
                                     cp.KruskalModel(inst.factors), 0, mode, inst.rho)
    assert p.set_operator("gram") == "gram"
    x = ri.random_matrix(inst.rng, shape[0] * r, 1).reshape(-1)
    assert ri.rel(cp.unaligned_matvec(p, x), orc.unaligned_matvec(inst.sub, x)) < 1e-12
    p.set_operator("stream")
    assert ri.rel(cp.unaligned_matvec(p, x), orc.unaligned_matvec(inst.sub, x)) < 1e-12


def test_gram_split_rows_and_empty_rows(cp):
    """One huge row (split over many CTAs by the partition planner) plus empty rows."""
    g = cp.Mt19937_64(5)
    shape = [40, 30, 20]
    r = 16
    factors = ri.random_model(shape, r, g)
    rs = np.random.default_rng(3)
    q = 400_000
    i0 = np.where(rs.random(q) < 0.7, 3, rs.integers(0, 40, q))  # row 3 holds ~70 % of the draws
    i0[i0 == 17] = 18                                             # row 17 empty
    idx = np.stack([i0, rs.integers(0, 30, q), rs.integers(0, 20, q)]).astype(np.int32)
    vals = rs.normal(size=q)
    mode = cp.RkhsMode(np.linspace(0, 1, 40), 0.1, 1e-3)
    kern = mode.kernel()
    p = cp.make_unaligned_subproblem(cp.ObservationSet(shape, idx, vals, multiset=True), cp.KruskalModel(factors), 0,
                                     mode, 1e-6)
    x = np.random.default_rng(4).normal(size=40 * r)
    y_o = orc.unaligned_matvec_stream(shape, 0, idx, factors, kern, 1e-3, 1e-6, x)
    assert ri.rel(cp.unaligned_matvec(p, x), y_o) < 1e-12
    p.set_operator("gram")
    assert ri.rel(cp.unaligned_matvec(p, x), y_o) < 1e-12
    assert ri.rel(p.b, orc.sampled_mttkrp_stream(shape, 0, idx, vals, factors, 40)) < 1e-12


def test_gram_auto_resolution(cp):
    c = ri.Inst([600, 8, 8], 4, 12000, 0, 0.5, 0.1, 1e-6, 7)  # n > 512, 20 obs / row >= 2 * rp = 8 -> gram
    mode = cp.RkhsMode(c.points, c.sigma, c.lam)
    p = cp.make_unaligned_subproblem(cp.ObservationSet(c.shape, c.idx, c.vals), cp.KruskalModel(c.factors), 0, mode,
                                     c.rho)
    assert p.operator() == "gram"          # a new plan starts with AUTO's choice
    assert p.set_operator("stream") == "stream"
    assert p.set_operator("auto") == "gram"
    c1 = ri.Inst([10, 8, 8], 4, 600, 0, 0.5, 0.1, 1e-6, 7)   # small n: the single fused launch -> stream
    mode1 = cp.RkhsMode(c1.points, c1.sigma, c1.lam)
    p1 = cp.make_unaligned_subproblem(cp.ObservationSet(c1.shape, c1.idx, c1.vals), cp.KruskalModel(c1.factors), 0,
                                      mode1, c1.rho)
    assert p1.operator() == "stream" and p1.set_operator("auto") == "stream"
    c2 = ri.Inst([50, 8, 8], 4, 60, 0, 0.5, 0.1, 1e-6, 8)   # ~1 obs / row -> stream
    mode2 = cp.RkhsMode(c2.points, c2.sigma, c2.lam)
    p2 = cp.make_unaligned_subproblem(cp.ObservationSet(c2.shape, c2.idx, c2.vals), cp.KruskalModel(c2.factors), 0,
                                      mode2, c2.rho)
    assert p2.set_operator("auto") == "stream"


def test_gram_pcg_config1(cp):
    """Config 1 PCG with the row-Gram operator: iterations within +-1, residual <= 1e-8."""
    from inputs import configs
    c = configs.config1()
    mode = cp.RkhsMode(c.points, c.ell, c.lam)
    kern = mode.kernel()
    ek = orc.sym_eig(kern)
    mode.set_eig(ek.u, ek.d)
    model = cp.KruskalModel([np.zeros((c.shape[0], c.r))] + c.factors[1:])
    p = cp.make_unaligned_subproblem(cp.ObservationSet(c.shape, c.idx, c.vals), model, 0, mode, c.rho)
    sub = orc.make_unaligned_subproblem(c.shape, c.idx, c.vals, model.factors, 0, kern, c.lam, c.rho)
    ev = orc.sym_eig(sub.v)
    p.set_v_eig(ev.u, ev.d)
    assert p.set_operator("gram") == "gram"
    rep, orep = cp.SolveReport(), orc.SolveReport()
    w = cp.solve_unaligned_pcg(p, cp.PcgConfig(c.tol, c.max_iter), rep)
    orc.solve_unaligned_pcg(sub, orc.PcgConfig(c.tol, c.max_iter), ek, ev, report=orep)
    assert rep.converged and rep.relative_residual <= c.tol
    assert abs(rep.iterations - orep.iterations) <= 1
    rhs = (kern @ sub.b).reshape(-1, order="F")
    tr = np.linalg.norm(rhs - orc.unaligned_matvec(sub, w.reshape(-1, order="F"))) / np.linalg.norm(rhs)
    assert tr <= 10 * c.tol


@pytest.mark.parametrize("which,q", [("config3", 2_000_000), ("config4", 3_000_000)])
def test_gram_large_config_structure(cp, which, q):
    from inputs import configs
    cfg = getattr(configs, which)()
    ctx = cp.default_context()
    idx, vals = cp.synth_observations_device(cfg, ctx, q)
    hidx = idx.cpu().numpy()
    n, r = cfg.shape[0], cfg.r
    mode = cp.RkhsMode(cfg.points, cfg.ell, cfg.lam, ctx=ctx, kernel=cfg.kernel)
    kern = mode.kernel()
    obs = cp.DeviceObservations(cfg.shape, idx.data_ptr(), vals.data_ptr(), q, keepalive=(idx, vals))
    model = cp.KruskalModel([np.zeros((n, r))] + cfg.factors[1:])
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, cfg.rho)
    assert p.set_operator("gram") == "gram"
    x = np.random.default_rng(1).normal(size=n * r)
    y_o = orc.unaligned_matvec_stream(cfg.shape, 0, hidx, model.factors, kern, cfg.lam, cfg.rho, x)
    assert ri.rel(cp.unaligned_matvec(p, x), y_o) < 1e-12


@pytest.mark.parametrize("shape,r,multiset", [([48, 20, 16, 6], 32, False), ([40, 64, 30], 64, True), ([30, 50, 9], 16, True),
                                              ([700, 30, 20], 64, False), ([600, 9, 7, 5, 6], 16, True),
                                              ([520, 40, 36], 24, True)])
def test_gram_build_v1_vs_v2(cp, monkeypatch, shape, r, multiset):
    """Row-Gram build: the register-fragment kernel (v3, k_gram3.cu, the default for RP 16 / 32 / 64
    and 2..4 other modes), the 2x2 register-blocked DMMA kernel (v2) and the one-tile-per-fragment
    kernel (v1) against each other and the oracle — coalesced multiset plans included (entry weights
    = multiplicities), rows split over many units (small n: the last arrival sums the unit slots),
    k-steps straddling row ends."""
    g = cp.Mt19937_64(11 + r)
    factors = ri.random_model(shape, r, g)
    rs = np.random.default_rng(r)
    q = 60_000
    idx = np.stack([rs.integers(0, n, q) for n in shape]).astype(np.int32)
    vals = rs.normal(size=q)
    mode = cp.RkhsMode(np.linspace(0, 1, shape[0]), 0.1, 1e-3)
    kern = mode.kernel()
    x = np.random.default_rng(5).normal(size=shape[0] * r)
    ys = {}
    for v, env in (("v1", {"CPHIFI_GRAM3": "0", "CPHIFI_GRAM_V2": "0"}), ("v2", {"CPHIFI_GRAM3": "0", "CPHIFI_GRAM_V2": "1"}),
                   ("v3", {"CPHIFI_GRAM3": "1"})):
        for k, val in env.items():
            monkeypatch.setenv(k, val)
        p = cp.make_unaligned_subproblem(cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=multiset),
                                         cp.KruskalModel(factors), 0, mode, 1e-6)
        p.set_operator("gram")
        ys[v] = cp.unaligned_matvec(p, x)
        assert np.array_equal(ys[v], cp.unaligned_matvec(p, x))
        monkeypatch.delenv("CPHIFI_GRAM_V2", raising=False)
    y_o = orc.unaligned_matvec_stream(shape, 0, idx, factors, kern, 1e-3, 1e-6, x)
    assert ri.rel(ys["v2"], ys["v1"]) < 1e-13
    assert ri.rel(ys["v3"], ys["v1"]) < 1e-13
    assert ri.rel(ys["v3"], y_o) < 1e-12
