"""Host restatement (numpy) of the multi-GPU observation cut the C-ABI library makes on the device
(csrc/capi.cu: balanced_shard_cuts, shard_rows): which contiguous slice of the sorted observations
each rank keeps, and which rows of mode k it owns.  For callers that plan a job without a GPU and
for the CPU tests (tests/test_sharding.py, tests/test_dist_gloo.py); the device path never calls it.

The observations are sorted lexicographically by (i_k, other modes ascending) — the storage order
of the reference's ObservationSet (observations.hpp:27-41) — and rank s of S keeps draws
[cuts[s], cuts[s + 1]).  SURVEY §8e shards the observations; equal COUNTS are the wrong unit for a
skewed set (config 4's Zipf rows: 88 % of the draws sit in saturated rows that run as cheap GEMMs),
so the cut balances the modelled q-pass time instead."""
from __future__ import annotations

import math

import numpy as np

DENSE_MIN = 0.3               # build_dense_rows: a 3-way row this full runs as two DMMA GEMMs
DENSE_ROW_COST_CELLS = 0.345  # ... at the cost of this many plan entries per grid cell
RUN_COST_ENTRIES = 21.0       # per-run work of the run kernel, in entries


def sorted_keys(idx: np.ndarray, shape, k: int):
    """Lexicographic u64 keys (i_k most significant, then the other modes ascending), sorted; span =
    the product of the other mode sizes (row of a key = key // span)."""
    d = len(shape)
    stride, span = [0] * d, 1
    for m in range(d - 1, -1, -1):
        if m == k:
            continue
        stride[m] = span
        span *= int(shape[m])
    stride[k] = span
    keys = np.zeros(idx.shape[1], dtype=np.uint64)
    for m in range(d):
        keys += idx[m].astype(np.uint64) * np.uint64(stride[m])
    return np.sort(keys, kind="stable"), span


def shard_cuts(idx: np.ndarray, shape, k: int, shards: int, coalesce: bool, equal_count: bool = False,
               dense_min: float = DENSE_MIN, by_entries: bool = False):
    """(cuts, rp): the S + 1 cut positions in the sorted draws and the row pointers of all draws."""
    keys, span = sorted_keys(idx, shape, k)
    q, nk, d = keys.size, int(shape[k]), len(shape)
    rp = np.searchsorted(keys, np.arange(nk + 1, dtype=np.uint64) * np.uint64(span), side="left").astype(np.int64)
    cuts = [q * t // shards for t in range(shards + 1)]
    if equal_count or shards <= 1 or q == 0:
        return cuts, rp
    draws = np.diff(rp).astype(np.float64)
    if coalesce:
        first = np.ones(q, dtype=bool)
        first[1:] = keys[1:] != keys[:-1]
        ent = np.bincount((keys[first] // np.uint64(span)).astype(np.int64), minlength=nk).astype(np.float64)
    else:
        ent = draws
    n_first = float(shape[1 if k == 0 else 0])
    cost = ent if by_entries else ent + RUN_COST_ENTRIES * np.minimum(ent, n_first)
    if d == 3 and dense_min > 0.0 and not by_entries:
        cost = np.where(ent >= dense_min * float(span), DENSE_ROW_COST_CELLS * float(span), cost)
    pre = np.concatenate([[0.0], np.cumsum(cost)])  # the same left-to-right double sum as the host loop
    total = float(pre[nk])
    for t in range(1, shards):
        pos = q * t // shards
        if total > 0.0:
            target = total * float(t) / float(shards)
            i = int(np.searchsorted(pre, target, side="right")) - 1
            i = min(max(i, 0), nk - 1)
            ci = float(pre[i + 1] - pre[i])
            if ci <= total / (4.0 * shards):
                pos = int(rp[i]) if target - pre[i] < pre[i + 1] - target else int(rp[i + 1])
            else:
                pos = int(rp[i]) + int(math.floor((target - pre[i]) / ci * float(rp[i + 1] - rp[i]) + 0.5))
        cuts[t] = min(q, max(cuts[t - 1], pos))
    return cuts, rp


def shard_row_ranges(cuts, rp, shard: int):
    """(own_lo, own_hi, hull_hi), multiples of 8 rows: the rank owns rows [own_lo, own_hi) — a
    partition of [0, n_k) over the ranks — and its observations lie in rows [own_lo, hull_hi)."""
    nk, S = len(rp) - 1, len(cuts) - 1

    def first_row(t):
        if t <= 0:
            return 0
        if t >= S:
            return nk
        i = int(np.searchsorted(rp, cuts[t], side="right")) - 1
        return min(max(i, 0), nk) // 8 * 8

    own_lo = first_row(shard)
    own_hi = nk if shard + 1 >= S else first_row(shard + 1)
    hull_hi = nk if shard + 1 >= S else min(nk, own_hi + 8)
    return own_lo, own_hi, hull_hi
