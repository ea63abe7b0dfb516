"""GPU: every alternative implementation of a hot-path row agrees with the oracle and with its
siblings (selected by the library's CPHIFI_* switches, read per call or per plan):

  * MTTKRP v1 (cp.async, 8 warps) / v2 (16 warps) / v3 (tensor-map TMA ring), even and odd n0,
    partial row tiles and partial k chunks                      (tensor.hpp:174-182)
  * eigenbasis sandwich v1 (cp.async) / v2 (bulk-copy ring) / four DMMA GEMMs, for the decoupled
    solve and the preconditioner                                 (aligned.hpp:41-54, unaligned.hpp:135-139)
  * PCG device-resident CUDA-graph loop vs the host loop: identical iterates and history
    (solvers.hpp:38-88)
  * host-buffer matvec through the cached [copy in, operator, copy out] graph vs plain calls
  * equal-count vs row-aligned partition of the fused operator (split rows)

Tolerances: 1e-12 relative against the oracle (fp64 summation order only); bitwise equality
where two paths run the same arithmetic in the same order (PCG graph vs host loop).
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


@pytest.mark.parametrize("shape,r", [([200, 100, 60], 10), ([130, 34, 6], 32), ([64, 8, 6, 5], 16),
                                     ([37, 11, 9], 5), ([256, 64, 4], 8), ([150, 7], 3)])
def test_mttkrp_variants_vs_oracle(cp, monkeypatch, shape, r):
    g = cp.Mt19937_64(sum(shape) + r)
    flat = ri.random_tensor(shape, g)
    factors = ri.random_model(shape, r, g)
    t = cp.DenseTensor(shape, flat)
    bo = orc.mttkrp(flat.reshape(shape, order="F"), factors, 0)
    out = {}
    for v1, v3 in (("1", "0"), ("0", "0"), ("0", "1")):
        monkeypatch.setenv("CPHIFI_MTTKRP_V1", v1)
        monkeypatch.setenv("CPHIFI_MTTKRP_V3", v3)
        b = cp.mttkrp(t, cp.KruskalModel(factors), 0)
        assert ri.rel(b, bo) < 1e-12, (v1, v3)
        out[(v1, v3)] = b
    # every variant is deterministic: a second call is bit-identical
    b2 = cp.mttkrp(t, cp.KruskalModel(factors), 0)
    assert np.array_equal(b2, out[("0", "1")])


@pytest.mark.parametrize("n,r", [(200, 10), (64, 32), (130, 64), (33, 5), (300, 1), (1024, 32), (2048, 64)])
def test_decoupled_sandwich_variants(cp, monkeypatch, n, r):
    g = cp.Mt19937_64(7 * n + r)
    pts = np.sort(g.uniform_real(0, 1, n))
    mode = cp.RkhsMode(pts, 0.1, 1e-3)
    kern = mode.kernel()
    ek = orc.sym_eig(kern)
    mode.set_eig(ek.u, ek.d)
    b = ri.random_matrix(g, n, r)
    v = ri.random_spd(g, r)
    ev = orc.sym_eig(v)
    wo = orc.solve_aligned_decoupled(b, ek, ev, 1e-3)
    ws = {}
    for sw, v1, v3, v4, v5 in (("0", "0", "0", "0", "0"), ("1", "1", "0", "0", "0"), ("1", "0", "0", "0", "0"),
                               ("1", "0", "1", "0", "0"), ("1", "0", "1", "1", "0"), ("1", "0", "1", "0", "8"),
                               ("1", "0", "1", "0", "2")):
        monkeypatch.setenv("CPHIFI_SANDWICH", sw)
        monkeypatch.setenv("CPHIFI_SANDWICH_V1", v1)
        monkeypatch.setenv("CPHIFI_SANDWICH_V3", v3)  # v3: DMMA (even n >= 512)
        monkeypatch.setenv("CPHIFI_SANDWICH_V4", v4)  # v4: split-K DMMA (opt-in)
        monkeypatch.setenv("CPHIFI_SANDWICH_V5", v5)  # v5: v3 + cluster multicast (cap on the cluster size)
        w = cp.solve_aligned_decoupled(cp.AlignedSubproblem(b, v, mode), ev)
        assert ri.rel(w, wo) < 1e-11, (sw, v1, v3, v4, v5)
        ws[v5 if v3 == "1" and v4 == "0" else None] = w
    # v5 keeps v3's fragments and summation order: bit-identical
    assert np.array_equal(ws["8"], ws["0"]) and np.array_equal(ws["2"], ws["0"])
    # zero denominator through the mapped status word (sandwich path)
    monkeypatch.setenv("CPHIFI_SANDWICH", "1")
    mode0 = cp.RkhsMode(ri.identity_points(4), 1.0, 0.0)
    with pytest.raises(cp.CphifiRuntimeError, match="zero eigenvalue pair"):
        cp.solve_aligned_decoupled(cp.AlignedSubproblem(ri.random_matrix(g, 4, 2), np.zeros((2, 2)), mode0))


def _config1_problem(cp, shared=True):
    from inputs import configs
    c = configs.config1()
    n, r = c.shape[0], c.r
    mode = cp.RkhsMode(c.points, c.ell, c.lam)
    kern = mode.kernel()
    ek = orc.sym_eig(kern)
    if shared:
        mode.set_eig(ek.u, ek.d)
    model = cp.KruskalModel([np.zeros((n, r))] + c.factors[1:])
    p = cp.make_unaligned_subproblem(cp.ObservationSet(c.shape, c.idx, c.vals), model, 0, mode, c.rho)
    sub = orc.make_unaligned_subproblem(c.shape, c.idx, c.vals, model.factors, 0, kern, c.lam, c.rho)
    return c, p, sub, ek


def test_precond_sandwich_variants(cp, monkeypatch):
    c, p, sub, ek = _config1_problem(cp)
    ev = orc.sym_eig(sub.v)
    p.set_v_eig(ev.u, ev.d)
    x = np.random.default_rng(3).normal(size=c.shape[0] * c.r)
    yo = orc.build_preconditioner(sub, ek, ev).apply(x)
    for sw, v1, v3, v4, v5 in (("0", "0", "0", "0", "0"), ("1", "1", "0", "0", "0"), ("1", "0", "0", "0", "0"),
                               ("1", "0", "1", "0", "0"), ("1", "0", "1", "1", "0"), ("1", "0", "1", "0", "8")):
        monkeypatch.setenv("CPHIFI_SANDWICH", sw)
        monkeypatch.setenv("CPHIFI_SANDWICH_V1", v1)
        monkeypatch.setenv("CPHIFI_SANDWICH_V3", v3)
        monkeypatch.setenv("CPHIFI_SANDWICH_V4", v4)
        monkeypatch.setenv("CPHIFI_SANDWICH_V5", v5)
        y = cp.build_preconditioner(p).apply(x)
        assert ri.rel(y, yo) < 1e-12, (sw, v1, v3, v4, v5)


def test_pcg_graph_loop_matches_host_loop(cp, monkeypatch):
    c, p, sub, ek = _config1_problem(cp)
    ev = orc.sym_eig(sub.v)
    p.set_v_eig(ev.u, ev.d)
    res = {}
    for gflag in ("0", "1", "1"):  # host loop, graph build, graph reuse
        monkeypatch.setenv("CPHIFI_PCG_GRAPH", gflag)
        rep = cp.SolveReport()
        w = cp.solve_unaligned_pcg(p, cp.PcgConfig(c.tol, c.max_iter, record_history=True), rep)
        res.setdefault(gflag, []).append((w, rep))
    (wh, rh), = res["0"]
    for wg, rg in res["1"]:
        assert np.array_equal(wg, wh)
        assert rg.iterations == rh.iterations and rg.residual_history == rh.residual_history
        assert rg.converged and rg.relative_residual <= c.tol
    # max_iter stops the device loop at exactly max_iter (solvers.hpp:59)
    monkeypatch.setenv("CPHIFI_PCG_GRAPH", "1")
    rep = cp.SolveReport()
    cp.solve_unaligned_pcg(p, cp.PcgConfig(1e-30, 3, record_history=True), rep)
    assert rep.iterations == 3 and len(rep.residual_history) == 4 and not rep.converged


def test_host_matvec_graph_vs_plain(cp, monkeypatch):
    import torch
    c, p, sub, ek = _config1_problem(cp, shared=False)
    n, r = c.shape[0], c.r
    xs = [torch.randn(n * r, dtype=torch.float64).pin_memory() for _ in range(2)]
    yo = [orc.unaligned_matvec(sub, x.numpy()) for x in xs]
    monkeypatch.setenv("CPHIFI_HOST_GRAPH", "1")
    for rep in range(2):  # second pass re-points the cached graph's copy nodes
        for x, ref in zip(xs, yo):
            y = torch.empty(n * r, dtype=torch.float64).pin_memory()
            from paper_2603_25691_b200 import _capi
            _capi.call("cphifi_unaligned_matvec", p.handle, x.numpy().ctypes.data_as(_capi.c_double_p),
                       y.numpy().ctypes.data_as(_capi.c_double_p))
            assert ri.rel(y.numpy(), ref) < 1e-12
    monkeypatch.setenv("CPHIFI_HOST_GRAPH", "0")
    y = cp.unaligned_matvec(p, xs[0].numpy())  # pageable path
    assert ri.rel(y, yo[0]) < 1e-12


@pytest.mark.parametrize("equal", ["148", "296", "7"])
def test_equal_partition_split_rows(cp, monkeypatch, equal):
    monkeypatch.setenv("CPHIFI_EQUAL_PART", equal)
    c, p, sub, ek = _config1_problem(cp, shared=False)
    x = np.random.default_rng(5).normal(size=c.shape[0] * c.r)
    assert ri.rel(cp.unaligned_matvec(p, x), orc.unaligned_matvec(sub, x)) < 1e-12


@pytest.mark.parametrize("op", ["stream", "gram"])
def test_pcg_eigenbasis_matches_original_basis(cp, monkeypatch, op):
    """PCG in the eigenbasis of K (large n: two n x n products per iteration instead of four) vs
    the reference-structured PCG and the oracle: iterations within +-1, residual <= tol, W within
    the solve tolerance (the clamped spectrum differs from K only at rounding level)."""
    g = np.random.default_rng(600)
    shape, r, q = [600, 30, 20], 8, 30000
    pts = np.sort(g.uniform(0, 1, shape[0]))
    lin = g.choice(int(np.prod(shape)), size=q, replace=False)
    idx = np.array(np.unravel_index(lin, shape, order="F"), dtype=np.int64)
    vals = g.normal(size=q)
    factors = [np.zeros((shape[0], r))] + [g.normal(size=(n, r)) for n in shape[1:]]
    mode = cp.RkhsMode(pts, 0.05, 1e-3)
    kern = mode.kernel()
    ek = orc.sym_eig(kern)
    mode.set_eig(ek.u, ek.d)
    p = cp.make_unaligned_subproblem(cp.ObservationSet(shape, idx, vals), cp.KruskalModel(factors), 0, mode, 1e-6)
    p.set_operator(op)
    cfg = cp.PcgConfig(1e-8, 500)
    out = {}
    for rot in ("0", "1"):
        monkeypatch.setenv("CPHIFI_PCG_EIGBASIS", rot)
        rep = cp.SolveReport()
        out[rot] = (cp.solve_unaligned_pcg(p, cfg, rep), rep)
    sub = orc.make_unaligned_subproblem(shape, idx, vals, factors, 0, kern, 1e-3, 1e-6)
    orep = orc.SolveReport()
    wo = orc.solve_unaligned_pcg(sub, orc.PcgConfig(1e-8, 500), ek, orc.sym_eig(sub.v), report=orep)
    for rot, (w, rep) in out.items():
        assert rep.converged and rep.relative_residual <= 1e-8, rot
        assert abs(rep.iterations - orep.iterations) <= 1, (rot, rep.iterations, orep.iterations)
        assert ri.rel(w, wo) < 1e-6, rot
    # warm start from the solution: converges at once in both bases
    for rot in ("0", "1"):
        monkeypatch.setenv("CPHIFI_PCG_EIGBASIS", rot)
        rep = cp.SolveReport()
        cp.solve_unaligned_pcg(p, cfg, rep, warm_start=out["0"][0])
        assert rep.iterations <= 1, rot


def test_mttkrp_v3_odd_rank_many_outer(cp, monkeypatch):
    """Odd r with several `outer` rows: the Khatri-Rao rows are 16-byte padded for the bulk copy."""
    g = cp.Mt19937_64(77)
    shape, r = [64, 40, 7], 5
    flat = ri.random_tensor(shape, g)
    factors = ri.random_model(shape, r, g)
    t = cp.DenseTensor(shape, flat)
    bo = orc.mttkrp(flat.reshape(shape, order="F"), factors, 0)
    for v1, v3 in (("1", "0"), ("0", "0"), ("0", "1")):
        monkeypatch.setenv("CPHIFI_MTTKRP_V1", v1)
        monkeypatch.setenv("CPHIFI_MTTKRP_V3", v3)
        assert ri.rel(cp.mttkrp(t, cp.KruskalModel(factors), 0), bo) < 1e-12, (v1, v3)


@pytest.mark.parametrize("fused,skipzero,graph", [("0", "0", "1"), ("1", "0", "1"), ("0", "1", "1"), ("1", "1", "1"),
                                                  ("1", "1", "0"), ("0", "1", "0")])
def test_pcg_large_n_step_variants(cp, monkeypatch, fused, skipzero, graph):
    """Large-n eigenbasis PCG: the one-launch cooperative vector step (k_pcgstep.cu) and the GEMMs
    that skip the clamped null space of K (mu_i = 0 rows / columns) against the oracle — each
    setting on a fresh plan (the captured solve graph bakes both in).  Residual history within
    1e-6 relative of the separate-kernel / full-GEMM path's (fp64 summation order only)."""
    g = np.random.default_rng(601)
    shape, r, q = [640, 24, 20], 12, 40000
    pts = np.sort(g.uniform(0, 1, shape[0]))
    lin = g.choice(int(np.prod(shape)), size=q, replace=False)
    idx = np.array(np.unravel_index(lin, shape, order="F"), dtype=np.int64)
    vals = g.normal(size=q)
    factors = [np.zeros((shape[0], r))] + [g.normal(size=(n, r)) for n in shape[1:]]
    mode = cp.RkhsMode(pts, 0.05, 1e-3)
    kern = mode.kernel()
    ek = orc.sym_eig(kern)
    assert (ek.d == 0).sum() >= 8  # the null-space skip is exercised
    mode.set_eig(ek.u, ek.d)
    cfg = cp.PcgConfig(1e-9, 500, record_history=True)
    res = {}
    for f, z, gr in (("0", "0", "1"), (fused, skipzero, graph)):
        monkeypatch.setenv("CPHIFI_PCG_FUSED", f)
        monkeypatch.setenv("CPHIFI_PCG_SKIPZERO", z)
        monkeypatch.setenv("CPHIFI_PCG_GRAPH", gr)  # "0" + fused: the speculative host loop
        p = cp.make_unaligned_subproblem(cp.ObservationSet(shape, idx, vals), cp.KruskalModel(factors), 0, mode, 1e-6)
        p.set_operator("gram")
        rep = cp.SolveReport()
        res[(f, z, gr)] = (cp.solve_unaligned_pcg(p, cfg, rep), rep)
    (w0, r0), (w1, r1) = res[("0", "0", "1")], res[(fused, skipzero, graph)]
    sub = orc.make_unaligned_subproblem(shape, idx, vals, factors, 0, kern, 1e-3, 1e-6)
    orep = orc.SolveReport()
    wo = orc.solve_unaligned_pcg(sub, orc.PcgConfig(1e-9, 500), ek, orc.sym_eig(sub.v), report=orep)
    assert r1.converged and r1.relative_residual <= 1e-9
    assert abs(r1.iterations - orep.iterations) <= 1, (r1.iterations, orep.iterations)
    assert r1.iterations == r0.iterations
    h0, h1 = np.asarray(r0.residual_history), np.asarray(r1.residual_history)
    assert h0.size == h1.size and np.all(np.abs(h1 - h0) <= 1e-6 * h0), (h0, h1)
    assert ri.rel(w1, w0) < 1e-9 and ri.rel(w1, wo) < 1e-6


def test_pcg_gram_epilogue_bitwise(cp, monkeypatch):
    """Large-n eigenbasis PCG with the row-Gram operator: the split-K reduction fused with the
    row-Gram apply (EPI_GRAM, one launch) sums in the same order as the two launches it replaces,
    so the solve is bit-identical; and it matches the oracle."""
    g = np.random.default_rng(602)
    shape, r, q = [1100, 20, 16], 16, 30000
    pts = np.sort(g.uniform(0, 1, shape[0]))
    lin = g.choice(int(np.prod(shape)), size=q, replace=False)
    idx = np.array(np.unravel_index(lin, shape, order="F"), dtype=np.int64)
    vals = g.normal(size=q)
    factors = [np.zeros((shape[0], r))] + [g.normal(size=(n, r)) for n in shape[1:]]
    mode = cp.RkhsMode(pts, 0.3, 1e-3)
    kern = mode.kernel()
    ek = orc.sym_eig(kern)
    mode.set_eig(ek.u, ek.d)
    assert shape[0] - (ek.d == 0).sum() >= 520  # the GEMM keeps k >= 512: tensor-map path with EPI_GRAM
    cfg = cp.PcgConfig(1e-9, 300, record_history=True)
    res = {}
    for epi in ("0", "1", "parts"):  # "parts": + the output GEMM's split-K partials reduced in the step
        monkeypatch.setenv("CPHIFI_GRAM_EPI", "0" if epi == "0" else "1")
        monkeypatch.setenv("CPHIFI_PCG_AP_PARTS", "1" if epi == "parts" else "0")
        p = cp.make_unaligned_subproblem(cp.ObservationSet(shape, idx, vals), cp.KruskalModel(factors), 0, mode, 1e-6)
        p.set_operator("gram")
        rep = cp.SolveReport()
        res[epi] = (cp.solve_unaligned_pcg(p, cfg, rep), rep)
    (w0, r0), (w1, r1) = res["0"], res["1"]
    assert r1.iterations == r0.iterations and r1.residual_history == r0.residual_history
    assert np.array_equal(w0, w1)
    w2, r2 = res["parts"]  # same sums; the epilogue's FMA contraction may differ by an ulp
    assert r2.iterations == r0.iterations and ri.rel(w2, w0) < 1e-10
    sub = orc.make_unaligned_subproblem(shape, idx, vals, factors, 0, kern, 1e-3, 1e-6)
    orep = orc.SolveReport()
    wo = orc.solve_unaligned_pcg(sub, orc.PcgConfig(1e-9, 300), ek, orc.sym_eig(sub.v), report=orep)
    assert r1.converged and abs(r1.iterations - orep.iterations) <= 1, (r1.iterations, orep.iterations)
    assert ri.rel(w1, wo) < 1e-6


def test_host_matvec_pinned_dma_vs_device(cp):
    """Large x / y in pinned host memory take the DMA path (cudaMemcpyAsync from / to the caller's
    buffers around an operator-only graph, no host staging copy): bit-identical to the device call,
    and re-captured when the operator form changes (stream -> gram)."""
    import torch
    from paper_2603_25691_b200 import _capi
    g = np.random.default_rng(3)
    shape, r, q = (4096, 64, 48), 32, 400000  # n r = 131072 doubles = 1 MB: the DMA path
    idx = np.stack([g.integers(0, s, q) for s in shape]).astype(np.int32)
    obs = cp.ObservationSet(shape, idx, g.normal(size=q), multiset=True, coalesce=True)
    mode = cp.RkhsMode(np.linspace(0, 1, shape[0]), 0.1, 1e-4)
    p = cp.make_unaligned_subproblem(obs, cp.KruskalModel([np.zeros((shape[0], r))] +
                                                          [g.normal(size=(s, r)) for s in shape[1:]]), 0, mode, 1e-6)
    n = shape[0]
    for op in ("stream", "gram", "stream"):
        p.set_operator(op)
        x = torch.randn(n * r, dtype=torch.float64).pin_memory()
        y = torch.empty(n * r, dtype=torch.float64).pin_memory()
        _capi.call("cphifi_unaligned_matvec", p.handle, x.numpy().ctypes.data_as(_capi.c_double_p),
                   y.numpy().ctypes.data_as(_capi.c_double_p))
        xd, yd = x.cuda(), torch.empty(n * r, dtype=torch.float64, device="cuda")
        _capi.call("cphifi_unaligned_matvec_device", p.handle, xd.data_ptr(), yd.data_ptr())
        torch.cuda.synchronize()
        assert torch.equal(y, yd.cpu()), op
