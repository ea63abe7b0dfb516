"""The run kernel (k_runs.cu: the operator's q-pass over a run table, per-warp TMA rings, factors
staged in shared memory, factor-block parts when they do not fit) against the oracle's streaming
restatement (observations.hpp:174-198) and against the previous streaming kernel (CPHIFI_RUNS=0),
on shapes that reach every branch: d = 3 / 4 / 5, padded ranks 16 / 32 / 64, multiset plans with
coalesced multiplicities, one part or several (the last mode's factor cut into row blocks), rows
split between warps, empty rows."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _case(shape, r, q, seed, coalesce, zipf=False):
    import paper_2603_25691_b200 as cp
    g = np.random.default_rng(seed)
    n = shape[0]
    idx = np.stack([g.integers(0, s, q) for s in shape]).astype(np.int32)
    if zipf:  # a heavy head row and empty rows
        idx[0] = np.minimum((g.pareto(1.1, q) * 3).astype(np.int64), n - 1) // 2 * 2
    vals = g.normal(size=q)
    factors = [g.normal(size=(s, r)) for s in shape]
    pts = np.sort(g.uniform(size=n))
    mode = cp.RkhsMode(pts, 0.05, 1e-4)
    obs = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    model = cp.KruskalModel([np.zeros((n, r))] + factors[1:])
    return cp, mode, obs, model, idx, vals, factors


@pytest.mark.parametrize("shape,r,q,coalesce,zipf", [
    ((700, 40, 30), 16, 30000, False, False),
    ((700, 40, 30), 16, 30000, True, True),
    ((1100, 24, 20, 12), 32, 60000, False, True),
    ((600, 50, 256), 64, 80000, True, False),      # A_3: 256 x 64 x 8 B = 128 KB -> one part
    ((600, 64, 512), 64, 120000, True, True),      # A_3: 512 rows -> two row-block parts
    ((600, 60, 900), 32, 90000, False, False),     # A_3: 900 x 32 x 8 B = 225 KB -> parts
    ((520, 6, 5, 4, 7), 16, 20000, True, False),   # d = 5
])
def test_runs_kernel_vs_oracle_and_stream(monkeypatch, shape, r, q, coalesce, zipf):
    cp, mode, obs, model, idx, vals, factors = _case(shape, r, q, 7, coalesce, zipf)
    n = shape[0]
    xhat = np.asfortranarray(np.random.default_rng(1).normal(size=(n, r)))
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    p.set_operator("stream")
    y_runs = p.scatter_gather(xhat)
    y_orc = orc.scatter_gather_stream(shape, 0, idx, [None] + factors[1:], xhat)
    assert np.linalg.norm(y_runs - y_orc) / np.linalg.norm(y_orc) < 1e-12
    x = np.random.default_rng(2).normal(size=n * r)
    ya = cp.unaligned_matvec(p, x)
    assert np.array_equal(ya, cp.unaligned_matvec(p, x))  # bit-reproducible
    monkeypatch.setenv("CPHIFI_RUNS", "0")
    obs2 = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    p2 = cp.make_unaligned_subproblem(obs2, model, 0, mode, 1e-6)
    p2.set_operator("stream")
    yb = cp.unaligned_matvec(p2, x)
    assert np.linalg.norm(ya - yb) / np.linalg.norm(yb) < 1e-12
    # the RHS B (built by the streaming kernel with the values) and V are unaffected
    assert np.linalg.norm(p.b - p2.b) / np.linalg.norm(p2.b) < 1e-13


@pytest.mark.parametrize("shape,r,q,coalesce,zipf", [
    ((700, 40, 30), 16, 30000, False, False),
    ((1100, 24, 20, 12), 32, 60000, False, True),
    ((600, 64, 512), 64, 120000, True, True),      # two factor-block parts: G accumulated over launches
    ((600, 60, 900), 32, 90000, True, False),
])
def test_gram_ws_build_vs_oracle(monkeypatch, shape, r, q, coalesce, zipf):
    """The warp-specialised row-Gram build (k_gramws.cu, over the run parts) gives the operator the
    oracle's streaming restatement gives, and the same G as the single-pass build (CPHIFI_GRAM_WS=0)."""
    monkeypatch.setenv("CPHIFI_GRAM_WS", "1")  # opt-in build (k_gramws.cu)
    cp, mode, obs, model, idx, vals, factors = _case(shape, r, q, 11, coalesce, zipf)
    n = shape[0]
    x = np.random.default_rng(4).normal(size=n * r)
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    assert p.set_operator("gram") == "gram"
    y_ws = cp.unaligned_matvec(p, x)
    p.set_operator("stream")
    y_st = cp.unaligned_matvec(p, x)
    assert np.linalg.norm(y_ws - y_st) / np.linalg.norm(y_st) < 1e-12
    monkeypatch.setenv("CPHIFI_GRAM_WS", "0")
    obs2 = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    p2 = cp.make_unaligned_subproblem(obs2, model, 0, mode, 1e-6)
    p2.set_operator("gram")
    y_v = cp.unaligned_matvec(p2, x)
    assert np.linalg.norm(y_ws - y_v) / np.linalg.norm(y_v) < 1e-12
    y_o = orc.unaligned_matvec_stream(shape, 0, idx, [None] + factors[1:], mode.kernel(), 1e-4, 1e-6, x)
    assert np.linalg.norm(y_ws - y_o) / np.linalg.norm(y_o) < 1e-12


@pytest.mark.parametrize("shape,r,q,coalesce,zipf,dense", [
    ((600, 50, 256), 64, 80000, True, False, "0"),     # one part (the plan itself)
    ((600, 64, 512), 64, 120000, True, True, "0"),     # two factor-block parts
    ((600, 60, 900), 32, 90000, False, False, "0"),    # parts without multiplicities
    ((300, 40, 512), 64, 900000, True, True, "0.3"),   # dense rows: their parts carry B's entries too
])
def test_rhs_over_parts_vs_oracle_and_stream(monkeypatch, shape, r, q, coalesce, zipf, dense):
    """The right-hand side B = sampled_mttkrp(observed values) (observations.hpp:186-188) through the
    run kernel over every part of the q-pass plan (weights = values, no dot) against the oracle's
    streaming restatement and against the streaming kernel (CPHIFI_RHS_PARTS=0)."""
    monkeypatch.setenv("CPHIFI_DENSE_MIN", dense)
    cp, mode, obs, model, idx, vals, factors = _case(shape, r, q, 13, coalesce, zipf)
    n = shape[0]
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    plan = p.qpass_plan()
    assert plan["parts"] >= 1
    if dense != "0":
        assert plan["dense_rows"] > 0
    b_orc = orc.sampled_mttkrp_stream(shape, 0, idx, vals, [None] + factors[1:], n)
    assert np.linalg.norm(p.b - b_orc) / np.linalg.norm(b_orc) < 1e-12
    monkeypatch.setenv("CPHIFI_RHS_PARTS", "0")
    obs2 = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    p2 = cp.make_unaligned_subproblem(obs2, model, 0, mode, 1e-6)
    assert np.linalg.norm(p.b - p2.b) / np.linalg.norm(p2.b) < 1e-13
