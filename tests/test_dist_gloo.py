"""N > 1 host logic on CPU (gloo, world_size 2), mirroring the GPU path's multi-GPU scheme:
observations sorted by i_k and cut into contiguous equal-count shards [q*s/S, q*(s+1)/S), each
rank computes its partial Yhat, one all-reduce(sum) gives every rank the full Yhat and hence the
same operator output; the 128-byte NCCL id is distributed with broadcast_object_list the way
bench.py does it.  (The device kernels themselves are tested per shard on one GPU in
tests/test_gpu_parity.py::test_sharded_plans_sum_to_full.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from tests import refinst as ri
        inst = ri.Inst([30, 7, 6], 5, 800, 0, 0.6, 0.1, 1e-6, 2024)
        order = np.argsort(inst.idx[0], kind="stable")
        idx, vals = inst.idx[:, order], inst.vals[order]
        q = idx.shape[1]
        lo, hi = q * rank // world, q * (rank + 1) // world
        xhat = np.asfortranarray(np.random.default_rng(7).normal(size=(30, 5)))
        part = orc.scatter_gather_stream(inst.shape, 0, idx[:, lo:hi], inst.factors, xhat, threads=1)
        t = torch.from_numpy(np.ascontiguousarray(part).copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        full = orc.scatter_gather_stream(inst.shape, 0, idx, inst.factors, xhat, threads=1)
        err = float(np.linalg.norm(t.numpy() - full) / np.linalg.norm(full))
        # RHS B: sum of the shards' sampled MTTKRPs
        bp = torch.from_numpy(orc.sampled_mttkrp_stream(inst.shape, 0, idx[:, lo:hi], vals[lo:hi], inst.factors, 30,
                                                        threads=1).copy())
        dist.all_reduce(bp, op=dist.ReduceOp.SUM)
        berr = float(np.linalg.norm(bp.numpy() - inst.sub.b) / np.linalg.norm(inst.sub.b))
        # unique-id distribution (bench.py): rank 0's 128 bytes reach every rank
        uid = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        # max-over-ranks timing reduction
        tm = torch.tensor([float(rank + 1)])
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        out_q.put((rank, err, berr, uid[0] == bytes(range(128)), float(tm[0])))
    finally:
        dist.destroy_process_group()


def test_sharded_operator_allreduce_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, berr, uid_ok, tmax in res:
        assert err < 1e-12, (rank, err)
        assert berr < 1e-12, (rank, berr)
        assert uid_ok
        assert tmax == float(world)


def _als_worker(rank, world, port, out_q):
    """The ALS terms' multi-GPU scheme (capi.cu cphifi_als_update_*): every rank holds an equal-count
    shard of the i_k-sorted observations; the squared fit and ||v||^2 are summed over ranks
    (all-reduce of 2 scalars), the finite-mode row Grams G_i and right-hand sides B are summed
    (all-reduce of n x r x r and n x r) before the per-row solves — identical to the unsharded
    quantities."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = np.random.default_rng(11)
        shape, r, q, k = [9, 7, 6], 3, 240, 1
        lin = g.choice(int(np.prod(shape)), size=q, replace=False)
        idx = np.array(np.unravel_index(lin, shape, order="F"), dtype=np.int64)
        vals = g.normal(size=q)
        fac = [g.normal(size=(n, r)) for n in shape]
        order = np.argsort(idx[k], kind="stable")
        idx, vals = idx[:, order], vals[order]
        lo, hi = q * rank // world, q * (rank + 1) // world
        z = np.ones((q, r))
        for m in range(3):
            if m != k:
                z = z * fac[m][idx[m]]
        fit = np.einsum("lr,lr->l", z, fac[k][idx[k]])
        terms = torch.tensor([float(((vals[lo:hi] - fit[lo:hi]) ** 2).sum()), float((vals[lo:hi] ** 2).sum())],
                             dtype=torch.float64)
        dist.all_reduce(terms, op=dist.ReduceOp.SUM)
        rel = float(np.sqrt(terms[0]) / np.sqrt(terms[1]))
        rel_full = float(np.linalg.norm(vals - fit) / np.linalg.norm(vals))
        gsh = np.zeros((shape[k], r, r))
        bsh = np.zeros((shape[k], r))
        for l in range(lo, hi):
            gsh[idx[k, l]] += np.outer(z[l], z[l])
            bsh[idx[k, l]] += vals[l] * z[l]
        gt, bt = torch.from_numpy(gsh), torch.from_numpy(bsh)
        dist.all_reduce(gt, op=dist.ReduceOp.SUM)
        dist.all_reduce(bt, op=dist.ReduceOp.SUM)
        worst = 0.0
        for i in range(shape[k]):
            sel = np.nonzero(idx[k] == i)[0]
            if sel.size:
                ref = np.linalg.lstsq(z[sel], vals[sel], rcond=None)[0]
                ai = np.linalg.pinv(gt.numpy()[i]) @ bt.numpy()[i]
                worst = max(worst, float(np.linalg.norm(ai - ref) / np.linalg.norm(ref)))
        out_q.put((rank, abs(rel - rel_full) / rel_full, worst))
    finally:
        dist.destroy_process_group()


def test_sharded_als_terms_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_als_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rel_err, row_err in res:
        assert rel_err < 1e-13, (rank, rel_err)
        assert row_err < 1e-9, (rank, row_err)


def _row_sharded_worker(rank, world, port, out_q):
    """The row-sharded operator's multi-GPU scheme (capi.cu xhat_gemm_rows / y_gemm_rows) on CPU:
    cost-balanced row-aligned shards (paper_2603_25691_b200/sharding.py, the host restatement of
    the device cut), each rank contracts only its rows of K — Xhat[rows,:] = K[rows,:] X, its
    shard's partial Yhat, y_s = K[:, rows](Yhat_s[rows,:] + lambda X[owned rows,:]) (+ rho x on rank
    0) — and ONE all-reduce of the n x r partials gives the reference operator (unaligned.hpp:101-115)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc
        from paper_2603_25691_b200 import sharding
        from tests import refinst as ri
        inst = ri.Inst([40, 7, 6], 5, 900, 0, 0.6, 0.1, 1e-6, 77)
        n, r = 40, 5
        keys = (inst.idx[0].astype(np.int64) * 7 + inst.idx[1]) * 6 + inst.idx[2]
        order = np.argsort(keys, kind="stable")
        idx = inst.idx[:, order]
        cuts, rp = sharding.shard_cuts(inst.idx, inst.shape, 0, world, coalesce=False)
        lo, hi = cuts[rank], cuts[rank + 1]
        own_lo, own_hi, hull_hi = sharding.shard_row_ranges(cuts, rp, rank)
        x = np.random.default_rng(5).normal(size=n * r)
        xm = x.reshape(r, n).T  # column-major n x r
        kern = inst.kernel
        xhat = np.zeros((n, r))
        xhat[own_lo:hull_hi] = kern[own_lo:hull_hi, :] @ xm  # only this rank's rows of Xhat
        yhat = orc.scatter_gather_stream(inst.shape, 0, idx[:, lo:hi], inst.factors, np.asfortranarray(xhat), threads=1)
        assert not np.any(yhat[:own_lo]) and not np.any(yhat[hull_hi:])  # the shard touches only its rows
        op = yhat[own_lo:hull_hi].copy()
        op[:own_hi - own_lo] += inst.lam * xm[own_lo:own_hi]
        y_s = kern[:, own_lo:hull_hi] @ op
        if rank == 0:
            y_s = y_s + inst.rho * xm
        t = torch.from_numpy(np.ascontiguousarray(y_s))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        ref = orc.unaligned_matvec(inst.sub, x).reshape(r, n).T
        err = float(np.linalg.norm(t.numpy() - ref) / np.linalg.norm(ref))
        out_q.put((rank, err, (own_lo, own_hi, hull_hi), hi - lo))
    finally:
        dist.destroy_process_group()


def test_row_sharded_operator_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_row_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, rows, cnt in res:
        assert err < 1e-12, (rank, err)
        assert cnt > 0
    assert res[0][2][0] == 0 and res[0][2][1] == res[1][2][0] and res[1][2][1] == 40  # owned rows partition [0, n)
    assert sum(c for _, _, _, c in res) == 900
