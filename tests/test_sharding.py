"""The multi-GPU observation cut (paper_2603_25691_b200/sharding.py, the host restatement of
capi.cu's balanced_shard_cuts / shard_rows): properties on CPU, and the device cut against it."""
import ctypes

import numpy as np
import pytest

from paper_2603_25691_b200 import sharding


def _skewed(d3=True, n=640, q=300_000, seed=5):
    rng = np.random.default_rng(seed)
    shape = [n, 48, 40] if d3 else [n, 12, 10, 8]
    pz = 1.0 / np.arange(1, n + 1) ** 1.1
    i0 = rng.choice(n, size=q, p=pz / pz.sum())
    idx = np.stack([i0] + [rng.integers(0, s, size=q) for s in shape[1:]]).astype(np.int32)
    return shape, idx


@pytest.mark.parametrize("d3", [True, False])
@pytest.mark.parametrize("coalesce", [True, False])
@pytest.mark.parametrize("S", [2, 3, 8])
def test_cuts_partition_rows_and_balance(S, coalesce, d3):
    shape, idx = _skewed(d3)
    q, n = idx.shape[1], shape[0]
    cuts, rp = sharding.shard_cuts(idx, shape, 0, S, coalesce)
    assert cuts[0] == 0 and cuts[-1] == q and all(a <= b for a, b in zip(cuts, cuts[1:]))
    if d3:  # the head rows are dense (capped cost): no row exceeds a quarter shard, every cut is row-aligned
        assert all(c in set(rp.tolist()) for c in cuts)
    own = [sharding.shard_row_ranges(cuts, rp, s) for s in range(S)]
    assert own[0][0] == 0 and own[-1][1] == n
    for s in range(S):
        lo, hi, hull = own[s]
        assert lo % 8 == 0 and (hi % 8 == 0 or hi == n) and lo <= hi <= hull <= n
        if s + 1 < S:
            assert own[s + 1][0] == hi  # owned rows partition [0, n)
        if cuts[s + 1] > cuts[s]:  # the shard's observations lie inside [own_lo, hull_hi)
            r0 = int(np.searchsorted(rp, cuts[s], side="right")) - 1
            r1 = int(np.searchsorted(rp, cuts[s + 1] - 1, side="right")) - 1
            assert lo <= r0 and r1 < hull
    # modelled cost per shard within 15 % of the mean (row granularity), where equal counts are far off
    keys, span = sharding.sorted_keys(idx, shape, 0)

    def shard_cost(c):
        out = []
        for s in range(S):
            kk = keys[c[s]:c[s + 1]]
            rows = (kk // np.uint64(span)).astype(np.int64)
            ent = np.bincount(rows[np.r_[True, kk[1:] != kk[:-1]]] if coalesce else rows, minlength=n).astype(float)
            cost = ent + sharding.RUN_COST_ENTRIES * np.minimum(ent, shape[1])
            if d3:
                cost = np.where(ent >= 0.3 * span, sharding.DENSE_ROW_COST_CELLS * span, cost)
            out.append(cost.sum())
        return np.array(out)

    bal = shard_cost(cuts)
    assert bal.max() <= 1.15 * bal.mean()
    eq, _ = sharding.shard_cuts(idx, shape, 0, S, coalesce, equal_count=True)
    assert eq == [q * t // S for t in range(S + 1)]


def test_cut_inside_a_dominant_row():
    """One row holding most of the (uncoalesced, 4-way) observations is cut inside, by draw count."""
    rng = np.random.default_rng(1)
    shape, q = [16, 6, 5, 4], 20_000
    i0 = np.where(rng.uniform(size=q) < 0.9, 3, rng.integers(0, 16, size=q))
    idx = np.stack([i0] + [rng.integers(0, s, size=q) for s in shape[1:]]).astype(np.int32)
    cuts, rp = sharding.shard_cuts(idx, shape, 0, 4, coalesce=False)
    inside = [c for c in cuts[1:-1] if rp[3] < c < rp[4]]
    assert len(inside) >= 2
    sizes = np.diff(cuts)
    assert sizes.max() <= 1.2 * sizes.mean()


def test_by_entries_balances_plan_entries():
    """The row-Gram build's cut: plan entries (distinct cells) per shard within a row of equal."""
    shape, idx = _skewed(True)
    keys, _ = sharding.sorted_keys(idx, shape, 0)
    cuts, rp = sharding.shard_cuts(idx, shape, 0, 8, coalesce=True, by_entries=True)
    ent = np.array([np.unique(keys[cuts[s]:cuts[s + 1]]).size for s in range(8)], dtype=float)
    assert ent.max() <= 1.1 * ent.mean()
    cuts_t, _ = sharding.shard_cuts(idx, shape, 0, 8, coalesce=True)
    ent_t = np.array([np.unique(keys[cuts_t[s]:cuts_t[s + 1]]).size for s in range(8)], dtype=float)
    assert ent_t.max() > 1.5 * ent_t.mean()  # the q-pass-time cut gives the dense head rows' ranks more entries


@pytest.mark.gpu
@pytest.mark.parametrize("by_entries", [False, True])
@pytest.mark.parametrize("d3", [True, False])
@pytest.mark.parametrize("coalesce", [True, False])
@pytest.mark.parametrize("S", [3, 8])
def test_device_cut_matches_host(ctx, S, coalesce, d3, by_entries):
    import paper_2603_25691_b200 as cp
    from paper_2603_25691_b200 import _capi
    lib = _capi.load()
    shape, idx = _skewed(d3)
    vals = np.random.default_rng(2).normal(size=idx.shape[1])
    cuts, rp = sharding.shard_cuts(idx, shape, 0, S, coalesce, by_entries=by_entries)
    keys, _ = sharding.sorted_keys(idx, shape, 0)
    obs = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
    obs.shard_by_entries = by_entries
    for s in range(S):
        h = obs.plan(0, ctx, s, S).h
        qt, ql = ctypes.c_int64(), ctypes.c_int64()
        _capi.check(lib.cphifi_obs_info(h, ctypes.byref(qt), ctypes.byref(ql), None))
        kk = keys[cuts[s]:cuts[s + 1]]
        assert ql.value == (np.unique(kk).size if coalesce else kk.size)
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _capi.check(lib.cphifi_obs_shard_rows(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        assert (a.value, b.value, c.value) == sharding.shard_row_ranges(cuts, rp, s)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["tiny", "one_row", "more_shards_than_rows", "empty_rows"])
def test_device_cut_edge_cases(ctx, case):
    """Few observations, one occupied row, more shards than rows, long stretches of empty rows: the
    device cut equals the host restatement, the shards partition the observations, and the shards'
    partial results (row-sharded operator at n > 512) sum to the unsharded application."""
    import paper_2603_25691_b200 as cp
    from paper_2603_25691_b200 import _capi
    lib = _capi.load()
    rng = np.random.default_rng(9)
    n, S = 520, 4
    if case == "tiny":
        shape, q = [n, 5, 4], 5
        i0 = rng.integers(0, n, size=q)
    elif case == "one_row":
        shape, q = [n, 5, 4], 2000
        i0 = np.full(q, 77)
    elif case == "more_shards_than_rows":
        shape, q, S = [n, 6, 5], 600, 8
        i0 = rng.choice([3, 400, 519], size=q)
    else:
        shape, q = [n, 6, 5], 3000
        i0 = rng.choice(np.r_[0:4, 500:520], size=q)
    idx = np.stack([i0] + [rng.integers(0, s, size=q) for s in shape[1:]]).astype(np.int32)
    vals = rng.normal(size=q)
    r = 8
    factors = [np.asfortranarray(rng.normal(size=(s, r))) for s in shape]
    mode = cp.RkhsMode(np.sort(rng.uniform(size=n)), 0.05, 1e-3, ctx=ctx)
    model = cp.KruskalModel([np.zeros((n, r))] + factors[1:])
    x = rng.normal(size=n * r)
    for coalesce in (True, False):
        cuts, rp = sharding.shard_cuts(idx, shape, 0, S, coalesce)
        keys, _ = sharding.sorted_keys(idx, shape, 0)
        obs = cp.ObservationSet(shape, idx, vals, multiset=True, coalesce=coalesce)
        pref = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6)
        pref.set_operator("stream")
        yref = cp.unaligned_matvec(pref, x)
        ysum, total = np.zeros_like(yref), 0
        for s in range(S):
            h = obs.plan(0, ctx, s, S).h
            qt, ql = ctypes.c_int64(), ctypes.c_int64()
            _capi.check(lib.cphifi_obs_info(h, ctypes.byref(qt), ctypes.byref(ql), None))
            kk = keys[cuts[s]:cuts[s + 1]]
            assert ql.value == (np.unique(kk).size if coalesce else kk.size), (case, coalesce, s)
            total += kk.size
            a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            _capi.check(lib.cphifi_obs_shard_rows(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
            assert (a.value, b.value, c.value) == sharding.shard_row_ranges(cuts, rp, s)
            p = cp.make_unaligned_subproblem(obs, model, 0, mode, 1e-6, shard=s, shards=S)
            p.set_operator("stream")
            ysum += cp.unaligned_matvec(p, x)
        assert total == q
        assert np.linalg.norm(ysum - yref) <= 1e-12 * np.linalg.norm(yref), (case, coalesce)
