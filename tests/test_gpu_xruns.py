"""The cross-run q-pass kernel (k_xruns.cu: 3-way coalesced factor-block parts, runs padded to even
lengths, lane groups switching runs inside a step; opt-in, CPHIFI_XRUNS=1, measured slower at config
4) against the oracle's streaming restatement (observations.hpp:174-198) and against the default
run-at-a-time kernel (k_runs.cu) on the same plans: short runs (odd lengths padded, runs shorter than
a step), long runs, Zipf-headed rows split between warps, rows shorter than a step; and the row-Gram
builds over the padded parts (which must mask the run-start flags off the multiplicities)."""
import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _case(shape, r, q, seed, zipf):
    import paper_2603_25691_b200 as cp
    g = np.random.default_rng(seed)
    idx = np.stack([g.integers(0, s, q) for s in shape]).astype(np.int32)
    if zipf:  # a few heavy rows (split between warps) and a long sparse tail
        w = 1.0 / np.arange(1, shape[0] + 1) ** 1.1
        idx[0] = g.choice(shape[0], size=q, p=w / w.sum()).astype(np.int32)
    vals = g.normal(size=q)
    factors = [g.normal(size=(s, r)) for s in shape]
    obs = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=True)
    mode = cp.RkhsMode(np.linspace(0, 1, shape[0]), 0.1, 1e-4)
    model = cp.KruskalModel([np.zeros((shape[0], r))] + factors[1:])
    return cp, mode, obs, model, idx, vals, factors


@pytest.mark.parametrize("shape,r,q,zipf", [
    ((600, 64, 512), 64, 120000, True),    # A_2 512 rows: two parts; short runs (~2 per (i, a) per part)
    ((300, 40, 512), 64, 900000, True),    # long runs, heavy rows split between warps
    ((2000, 512, 512), 64, 60000, False),  # runs of length 1 (all padded), rows shorter than a step
])
def test_xruns_vs_oracle_and_runs(monkeypatch, shape, r, q, zipf):
    monkeypatch.setenv("CPHIFI_DENSE_MIN", "0")  # every row on the run kernels
    monkeypatch.setenv("CPHIFI_XRUNS", "1")
    cp, mode, obs, model, idx, vals, factors = _case(shape, r, q, 3, zipf)
    n = shape[0]
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    p.set_operator("stream")
    plan = p.qpass_plan()
    assert plan["parts"] == 2 and plan["xruns_parts"] == 2
    xhat = np.random.default_rng(1).normal(size=(n, r))
    y = p.scatter_gather(xhat)
    y_orc = orc.scatter_gather_stream(shape, 0, idx, [None] + factors[1:], xhat)
    assert np.linalg.norm(y - y_orc) <= 1e-12 * np.linalg.norm(y_orc)
    # the padding adds at most one entry per run; the draws are the plan's
    assert plan["sparse_draws"] == q

    monkeypatch.setenv("CPHIFI_XRUNS", "0")
    obs2 = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=True)
    p2 = cp.make_unaligned_subproblem(obs2, model, 0, mode, 1e-6)
    p2.set_operator("stream")
    assert p2.qpass_plan()["xruns_parts"] == 0
    y2 = p2.scatter_gather(xhat)
    assert np.linalg.norm(y - y2) <= 1e-13 * np.linalg.norm(y2)
    # the whole operator, through the stream path, against the oracle's operator
    x = np.random.default_rng(2).normal(size=n * r)
    yo = orc.unaligned_matvec_stream(shape, 0, idx, [np.zeros((n, r))] + factors[1:], mode.kernel(), 1e-4, 1e-6, x)
    assert np.linalg.norm(cp.unaligned_matvec(p, x) - yo) <= 1e-11 * np.linalg.norm(yo)


@pytest.mark.parametrize("env", ["CPHIFI_GRAM3_PARTS", "CPHIFI_GRAM_WS"])
def test_gram_builds_over_padded_parts(monkeypatch, env):
    """The row-Gram builds over the q-pass plan's parts read the padded parts' multiplicities with the
    run-start flag masked: the gram operator equals the stream operator."""
    monkeypatch.setenv("CPHIFI_DENSE_MIN", "0")
    monkeypatch.setenv("CPHIFI_XRUNS", "1")
    monkeypatch.setenv(env, "1")
    cp, mode, obs, model, idx, vals, factors = _case((600, 64, 512), 64, 120000, 5, True)
    n, r = 600, 64
    p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    assert p.qpass_plan()["xruns_parts"] == 2
    x = np.random.default_rng(4).normal(size=n * r)
    p.set_operator("stream")
    ys = cp.unaligned_matvec(p, x)
    p.set_operator("gram")
    yg = cp.unaligned_matvec(p, x)
    assert np.linalg.norm(yg - ys) <= 1e-12 * np.linalg.norm(ys)
