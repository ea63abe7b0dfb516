"""Dense rows of the stream operator's q-pass (k_dense_rows.cu: a row whose cells are mostly drawn
runs as two DMMA GEMMs over its multiplicity grid, S = (A_1 diag Xhat(i,:)) A_2', T = W o S,
P = T A_2, Yhat(i,c) = sum_a A_1(a,c) P(a,c)) against the oracle's streaming restatement
(observations.hpp:174-198) and against the same plan with the dense path off (CPHIFI_DENSE_MIN=0),
on shapes that reach every branch: padded ranks 16 / 32 / 64, grids padded to the 64 x 64 blocks
(n_1, n_2 not multiples of 64), multisets with and without coalescing, dense rows next to one
run-kernel part or several (A_2 cut into row blocks), and a plan whose rows are all dense."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _case(shape, r, q, seed, coalesce, head_rows, head_frac):
    import paper_2603_25691_b200 as cp
    g = np.random.default_rng(seed)
    n = shape[0]
    idx = np.stack([g.integers(0, s, q) for s in shape]).astype(np.int32)
    heavy = g.random(q) < head_frac  # a head of rows whose cells are (nearly) all drawn
    idx[0, heavy] = g.integers(0, head_rows, int(heavy.sum())) * 3 % n
    vals = g.normal(size=q)
    factors = [g.normal(size=(s, r)) for s in shape]
    pts = np.sort(g.uniform(size=n))
    mode = cp.RkhsMode(pts, 0.05, 1e-4)
    obs = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    model = cp.KruskalModel([np.zeros((n, r))] + factors[1:])
    return cp, mode, obs, model, idx, vals, factors


CASES = [
    # shape, r, q, coalesce, head rows, head fraction
    ((600, 100, 90), 10, 400000, True, 4, 0.8),    # rp 16, grid padded to 128 x 128
    ((600, 100, 90), 10, 400000, False, 4, 0.8),   # multiset without coalescing: W counts repeats
    ((600, 64, 128), 24, 400000, True, 6, 0.7),    # rp 32, exact blocks
    ((600, 70, 512), 64, 900000, True, 5, 0.85),   # rp 64, A_2 512 rows: two run-kernel parts
    ((520, 9, 11), 16, 400000, True, 520, 1.0),    # every row dense: no run-kernel entries
]


@pytest.mark.parametrize("shape,r,q,coalesce,head,frac", CASES)
def test_dense_rows_vs_oracle_and_runs(monkeypatch, shape, r, q, coalesce, head, frac):
    cp, mode, obs, model, idx, vals, factors = _case(shape, r, q, 5, coalesce, head, frac)
    n = shape[0]
    xhat = np.asfortranarray(np.random.default_rng(1).normal(size=(n, r)))
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    p.set_operator("stream")
    plan = p.qpass_plan()
    assert plan["dense_rows"] > 0, plan
    y = p.scatter_gather(xhat)
    y_orc = orc.scatter_gather_stream(shape, 0, idx, [None] + factors[1:], xhat)
    assert np.linalg.norm(y - y_orc) / np.linalg.norm(y_orc) < 1e-12
    # row by row, dense rows included (each row to 1e-12 of its own norm)
    nz = np.linalg.norm(y_orc, axis=1) > 0
    rel = np.linalg.norm(y - y_orc, axis=1)[nz] / np.linalg.norm(y_orc, axis=1)[nz]
    assert rel.max() < 1e-11
    assert np.all(y[~nz] == 0.0)
    x = np.random.default_rng(2).normal(size=n * r)
    ya = cp.unaligned_matvec(p, x)
    assert np.array_equal(ya, cp.unaligned_matvec(p, x))  # fixed summation order: bit-reproducible
    monkeypatch.setenv("CPHIFI_DENSE_MIN", "0")
    obs2 = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    p2 = cp.make_unaligned_subproblem(obs2, model, 0, mode, 1e-6)
    p2.set_operator("stream")
    assert p2.qpass_plan()["dense_rows"] == 0
    yb = cp.unaligned_matvec(p2, x)
    assert np.linalg.norm(ya - yb) / np.linalg.norm(yb) < 1e-12


def test_dense_rows_threshold_split():
    """The plan keeps the rows under the density threshold on the run kernel: entries of dense rows
    leave the run-kernel parts, the rest stay."""
    cp, mode, obs, model, idx, vals, factors = _case((600, 100, 90), 10, 400000, 5, True, 4, 0.8)
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    p.set_operator("stream")
    plan = p.qpass_plan()
    key = np.unique((idx[0].astype(np.int64) * 100 + idx[1]) * 90 + idx[2])  # distinct cells
    cells = np.bincount(key // 9000, minlength=600)
    dense = cells >= 0.3 * 100 * 90
    assert plan["dense_rows"] == int(dense.sum())
    assert plan["sparse_entries"] == int(cells[~dense].sum())


def test_dense_rows_pcg_matches_runs(monkeypatch):
    """A full PCG solve with dense rows in the plan converges like the run-kernel-only plan."""
    cp, mode, obs, model, idx, vals, factors = _case((600, 64, 128), 24, 400000, 5, True, 6, 0.7)
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    p.set_operator("stream")
    assert p.qpass_plan()["dense_rows"] > 0
    cfg = cp.PcgConfig(tol=1e-8, max_iter=500)
    rep1, rep2 = cp.SolveReport(), cp.SolveReport()
    w1 = cp.solve_unaligned_pcg(p, cfg, rep1)
    monkeypatch.setenv("CPHIFI_DENSE_MIN", "0")
    obs2 = cp.ObservationSet((600, 64, 128), idx, vals, multiset=True, coalesce=True)
    p2 = cp.make_unaligned_subproblem(obs2, model, 0, mode, 1e-6)
    p2.set_operator("stream")
    w2 = cp.solve_unaligned_pcg(p2, cfg, rep2)
    assert abs(rep1.iterations - rep2.iterations) <= 1
    assert np.linalg.norm(w1 - w2) / np.linalg.norm(w2) < 1e-6


@pytest.mark.parametrize("shape,r,q,coalesce,head,frac", [
    ((600, 300, 512), 64, 900000, True, 5, 0.85),   # factors 415 KB: the build runs over the factor-block parts
    ((600, 300, 512), 64, 600000, False, 0, 0.0),   # no dense rows: run-kernel parts only
])
@pytest.mark.parametrize("stage", ["1", "3"])  # 3: mode 0 hoisted per run (opt-in)
def test_gram_build_over_parts(monkeypatch, shape, r, q, coalesce, head, frac, stage):
    """The row-Gram build over the q-pass plan's parts (the default: k_gram3.cu, block staged, mode 0
    through L1; the dense rows' entries in their own parts) gives the operator the oracle gives and the
    default single-pass build gives."""
    monkeypatch.setenv("CPHIFI_GRAM3_PARTS", stage)
    cp, mode, obs, model, idx, vals, factors = _case(shape, r, q, 9, coalesce, max(head, 1), frac)
    n = shape[0]
    x = np.random.default_rng(4).normal(size=n * r)
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    assert p.set_operator("gram") == "gram"
    y3 = cp.unaligned_matvec(p, x)
    assert np.array_equal(y3, cp.unaligned_matvec(p, x))
    # the dense rows' parts built concurrently on the plan's second stream (opt-in) instead of after
    # the sparse ones on one stream: every G_i sums in the same order, bit-identical
    monkeypatch.setenv("CPHIFI_GRAM_CONCURRENT", "1")
    obs_s = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    p_s = cp.make_unaligned_subproblem(obs_s, model, 0, mode, 1e-6)
    p_s.set_operator("gram")
    assert np.array_equal(cp.unaligned_matvec(p_s, x), y3)
    monkeypatch.delenv("CPHIFI_GRAM_CONCURRENT")
    plan = p.qpass_plan()
    assert plan["parts"] == 2
    if frac > 0:
        assert plan["dense_rows"] > 0
    kern = mode.kernel()
    y_o = orc.unaligned_matvec_stream(shape, 0, idx, [np.zeros((n, r))] + factors[1:], kern, 1e-4, 1e-6, x)
    assert np.linalg.norm(y3 - y_o) / np.linalg.norm(y_o) < 1e-12
    monkeypatch.setenv("CPHIFI_GRAM3_PARTS", "0")
    obs2 = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    p2 = cp.make_unaligned_subproblem(obs2, model, 0, mode, 1e-6)
    p2.set_operator("gram")
    y1 = cp.unaligned_matvec(p2, x)
    assert np.linalg.norm(y3 - y1) / np.linalg.norm(y1) < 1e-13


def test_qpass_plan_shared_by_subproblems():
    """Subproblems on the same observation plan share its q-pass plan (built once): a second
    subproblem with fresh factors reports the same plan and applies the operator the oracle gives."""
    cp, mode, obs, model, idx, vals, factors = _case((600, 64, 128), 24, 400000, 5, True, 6, 0.7)
    n, r = 600, 24
    p1 = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    p1.set_operator("stream")
    plan1 = p1.qpass_plan()
    g = np.random.default_rng(3)
    f2 = [np.zeros((n, r))] + [f * (1 + 0.1 * g.normal(size=f.shape)) for f in factors[1:]]
    p2 = cp.make_unaligned_subproblem(obs, cp.KruskalModel(f2), 0, mode, 1e-6)
    p2.set_operator("stream")
    assert p2.qpass_plan() == plan1
    xh = np.asfortranarray(np.random.default_rng(1).normal(size=(n, r)))
    y2 = p2.scatter_gather(xh)
    y_o = orc.scatter_gather_stream((600, 64, 128), 0, idx, [None] + f2[1:], xh)
    assert np.linalg.norm(y2 - y_o) / np.linalg.norm(y_o) < 1e-12
    y1 = p1.scatter_gather(xh)  # the first subproblem's own factors still apply
    y1_o = orc.scatter_gather_stream((600, 64, 128), 0, idx, [None] + factors[1:], xh)
    assert np.linalg.norm(y1 - y1_o) / np.linalg.norm(y1_o) < 1e-12
