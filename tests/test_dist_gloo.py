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
