"""The multi-rank code paths, executed on ONE GPU through the virtual communicator
(cphifi_vcomm: S contexts, one host thread each, collectives = rank-order sums in place of NCCL).

Every `is_multi` branch of the C-ABI runs here: observation shards with the out-of-place Yhat
all-reduce per application (the two-launch fused split at small n, the GEMM + stream kernel +
all-reduce at large n), the B all-reduce at plan creation, the host-loop PCG with the fused vector
step, the all-shard row Grams of the finite-mode update, and the aligned MTTKRP over mode-1 slabs
with the B all-reduce (observations.hpp:174-198, tensor.hpp:174-182).  Results are
compared with the unsharded plan; all ranks must hold bit-identical iterates.
"""
import threading

import numpy as np
import pytest

from inputs import configs

pytestmark = pytest.mark.gpu


def run_ranks(S, fn, timeout=600):
    """fn(ctx, rank, S) on S threads, each with its own context joined to one virtual communicator."""
    import paper_2603_25691_b200 as cp
    vc = cp.VirtualComm(S)
    out, errs = [None] * S, []

    def work(rank):
        try:
            ctx = cp.Context(0)
            ctx.init_vcomm(vc, rank)
            out[rank] = fn(ctx, rank, S)
        except BaseException as e:  # noqa: BLE001 — reported below
            errs.append((rank, e))

    ts = [threading.Thread(target=work, args=(k,), daemon=True) for k in range(S)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not any(t.is_alive() for t in ts), "a rank hung in a collective"
    assert not errs, errs
    return out


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def _unaligned_case(c, ek, multiset):
    import paper_2603_25691_b200 as cp
    n, r = c.shape[0], c.r
    obs = cp.ObservationSet(c.shape, c.idx, c.vals, multiset=multiset)
    model = cp.KruskalModel([np.zeros((n, r))] + c.factors[1:])
    x = np.random.default_rng(11).normal(size=n * r)
    cfg = cp.PcgConfig(c.tol, c.max_iter, record_history=True)

    def solve(ctx, rank, S):
        mode = cp.RkhsMode(c.points, c.ell, c.lam, ctx=ctx, kernel=c.kernel)
        mode.set_eig(ek.u, ek.d)
        p = cp.make_unaligned_subproblem(obs, model, 0, mode, c.rho, shard=rank, shards=S)
        y = cp.unaligned_matvec(p, x)
        rep = cp.SolveReport()
        w = cp.solve_unaligned_pcg(p, cfg, rep)
        fin = cp.update_finite_mode_unaligned(obs, cp.KruskalModel([mode.kernel() @ w] + c.factors[1:]), 1, ctx=ctx,
                                              shard=rank, shards=S)
        return dict(y=y, b=p.b, w=w, it=rep.iterations, rel=rep.relative_residual, hist=rep.residual_history,
                    fin=fin, kmat=mode.kernel())

    return solve


def _check_unaligned(res, ref, S, w_tol):
    for k in range(1, S):  # replicated iterates: every rank holds the same bits
        assert np.array_equal(res[k]["y"], res[0]["y"])
        assert np.array_equal(res[k]["w"], res[0]["w"])
        assert res[k]["it"] == res[0]["it"]
    r0 = res[0]
    assert rel(r0["y"], ref["y"]) <= 1e-12
    assert rel(r0["b"], ref["b"]) <= 1e-12
    assert r0["it"] == ref["it"], (r0["it"], ref["it"])
    assert r0["rel"] <= 1e-8
    h0, hr = np.array(r0["hist"]), np.array(ref["hist"])
    assert np.max(np.abs(h0 - hr) / hr) <= 1e-6
    kmat = ref["kmat"]
    assert rel(kmat @ r0["w"], kmat @ ref["w"]) <= w_tol
    assert rel(r0["fin"], ref["fin"]) <= 1e-9


@pytest.mark.timeout(900)
@pytest.mark.parametrize("S", [2, 4])
def test_multirank_config1(ctx, S):
    """Config 1 (small n: the fused operator's two-launch split around the all-reduce)."""
    import paper_2603_25691_b200 as cp
    from oracle import oracle as orc
    c = configs.config1()
    ek = orc.sym_eig(orc.gaussian_kernel(c.points, c.ell))
    solve = _unaligned_case(c, ek, multiset=False)
    ref = solve(ctx, 0, 1)
    assert not ctx.world()[0] > 1
    res = run_ranks(S, solve)
    _check_unaligned(res, ref, S, w_tol=1e-7)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("S", [2, 4])
def test_multirank_config3_reduced_q(ctx, S):
    """Config 3's modes, kernel and factors with q = 4e6 draws (large n: K X GEMM, stream kernel on
    the shard, all-reduce, output GEMM; host-loop PCG with the fused vector step)."""
    from oracle import oracle as orc
    cfg = configs.config3()
    q = 4_000_000
    idx, vals = configs.generate_host(cfg, 0, q)
    c = configs.UnalignedConfig("config3q", cfg.shape, cfg.r, cfg.lam, cfg.rho, cfg.tol, cfg.max_iter, cfg.points,
                                cfg.kernel, cfg.ell, cfg.factors, cfg.w_true, idx, vals, multiset=True)
    ek = orc.sym_eig(orc.matern32_kernel(c.points, c.ell))
    solve = _unaligned_case(c, ek, multiset=True)
    ref = solve(ctx, 0, 1)
    res = run_ranks(S, solve)
    _check_unaligned(res, ref, S, w_tol=1e-6)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("S", [2, 4])
def test_multirank_aligned_config2(ctx, S):
    """Config 2's tensor sharded over mode-1 slabs: each rank's partial MTTKRP, B all-reduced."""
    import paper_2603_25691_b200 as cp
    c = configs.config2()
    t = cp.DenseTensor(c.shape, c.tensor)
    model = cp.KruskalModel([np.zeros((c.shape[0], c.r))] + c.factors[1:])
    ref = cp.mttkrp(t, model, 0, ctx)
    res = run_ranks(S, lambda cx, rank, S_: cp.mttkrp(t, model, 0, cx, shard=rank, shards=S_))
    for k in range(S):
        assert np.array_equal(res[k], res[0])
    assert rel(res[0], ref) <= 1e-12


def _skewed_case(d3: bool):
    """A Zipf-skewed multiset (the head rows saturate their grids, the tail is sparse), n = 640."""
    rng = np.random.default_rng(5)
    n, r = 640, 16
    shape = [n, 48, 40] if d3 else [n, 12, 10, 8]
    q = 300_000
    pz = 1.0 / np.arange(1, n + 1) ** 1.1
    i0 = rng.choice(n, size=q, p=pz / pz.sum())
    idx = np.stack([i0] + [rng.integers(0, s, size=q) for s in shape[1:]]).astype(np.int32)
    vals = rng.normal(size=q)
    pts = np.sort(rng.uniform(size=n))
    factors = [np.asfortranarray(rng.normal(size=(s, r))) for s in shape]
    return shape, r, idx, vals, pts, factors


@pytest.mark.parametrize("d3", [True, False])
@pytest.mark.parametrize("coalesce", [True, False])
@pytest.mark.parametrize("S", [2, 3, 8])
def test_balanced_shards_partials_sum(ctx, S, coalesce, d3):
    """Cost-balanced shards (capi.cu balanced_shard_cuts) and the row-sharded operator: with no
    communicator attached every shard returns its partial y_s = K[:, rows](Yhat_s + lambda X[owned])
    (+ rho x on shard 0); the partials of all shards sum to the unsharded application — for the
    balanced cut and the equal-count cut alike — and the cuts partition the observations."""
    import ctypes

    import paper_2603_25691_b200 as cp
    from paper_2603_25691_b200 import _capi
    shape, r, idx, vals, pts, factors = _skewed_case(d3)
    n, q = shape[0], vals.size
    mode = cp.RkhsMode(pts, 0.05, 1e-3, ctx=ctx)
    model = cp.KruskalModel([np.zeros((n, r))] + factors[1:])
    x = np.random.default_rng(3).normal(size=n * r)
    lib = _capi.load()

    def q_local(obs, s, S_):
        qt, ql = ctypes.c_int64(), ctypes.c_int64()
        _capi.check(lib.cphifi_obs_info(obs.plan(0, ctx, s, S_).h, ctypes.byref(qt), ctypes.byref(ql), None))
        return ql.value

    obs = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    pref = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
    pref.set_operator("stream")
    yref = cp.unaligned_matvec(pref, x)
    counts = {}
    for equal in (False, True):
        obs = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
        obs.equal_count_shards = equal
        ysum = np.zeros_like(yref)
        for s in range(S):
            p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6, shard=s, shards=S)
            p.set_operator("stream")
            ysum += cp.unaligned_matvec(p, x)
        assert rel(ysum, yref) <= 1e-12, (equal, rel(ysum, yref))
        counts[equal] = [q_local(obs, s, S) for s in range(S)]
    if not coalesce:
        assert sum(counts[False]) == q and sum(counts[True]) == q
        assert counts[True] == [q * (s + 1) // S - q * s // S for s in range(S)]
        # the skew: the balanced cut gives the saturated head rows' shard more draws than an equal share
        assert counts[False][0] > counts[True][0]
    else:
        assert sum(counts[False]) == q_local(cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=True), 0, 1)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("S", [3, 8])
def test_multirank_skewed_dense_rows(ctx, S):
    """The Zipf-skewed coalesced 3-way multiset under the virtual communicator: cost-balanced
    row-aligned shards (dense rows on the head ranks, sparse rows on the tail ranks), the
    row-sharded stream operator with its all-reduce of the n x r partial y, and the PCG solve on
    the sharded plan — against the unsharded plan; every rank holds the same bits."""
    import paper_2603_25691_b200 as cp
    shape, r, idx, vals, pts, factors = _skewed_case(True)
    n = shape[0]
    obs = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=True)
    model = cp.KruskalModel([np.zeros((n, r))] + factors[1:])
    x = np.random.default_rng(11).normal(size=n * r)
    cfg = cp.PcgConfig(1e-8, 500)

    def solve(cx, rank, S_):
        mode = cp.RkhsMode(pts, 0.05, 1e-3, ctx=cx)
        p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6, shard=rank, shards=S_)
        p.set_operator("stream")
        y = cp.unaligned_matvec(p, x)
        rep = cp.SolveReport()
        w = cp.solve_unaligned_pcg(p, cfg, rep)
        return dict(y=y, b=p.b, kw=mode.kernel() @ w, it=rep.iterations, rel=rep.relative_residual,
                    dense=p.qpass_plan()["dense_rows"])

    ref = solve(ctx, 0, 1)
    assert ref["dense"] > 0  # the head rows run as GEMMs
    res = run_ranks(S, solve)
    assert sum(o["dense"] for o in res) == ref["dense"]  # whole rows per rank: the single-GPU dense / sparse split
    for k in range(1, S):
        assert np.array_equal(res[k]["y"], res[0]["y"])
        assert np.array_equal(res[k]["kw"], res[0]["kw"])
    assert rel(res[0]["y"], ref["y"]) <= 1e-12
    assert rel(res[0]["b"], ref["b"]) <= 1e-12
    # ~135 iterations on this ill-conditioned multiset: the ranks' partial sums are added in another
    # order than the unsharded plan's, and the rounding drift moves the stopping iteration by a few
    assert abs(res[0]["it"] - ref["it"]) <= 4 and res[0]["rel"] <= 1e-8
    assert rel(res[0]["kw"], ref["kw"]) <= 1e-6
