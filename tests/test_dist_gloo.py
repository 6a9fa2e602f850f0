"""Multi-rank host plumbing on CPU (-m "not gpu"): frame sharding and the pa_step all-reduce
callback, world size 2 over gloo.  The per-rank compute here is the fp64 oracle acting as a
test double for libpa (test-only; the product path has no CPU fallback)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_09643_b200.dist import shard_frames


def test_shard_frames_partition_and_balance():
    for F in (0, 1, 5, 400, 801):
        for W in (1, 2, 3, 8):
            parts = [shard_frames(F, W, r) for r in range(W)]
            allf = np.sort(np.concatenate(parts)) if F else np.zeros(0)
            assert np.array_equal(allf, np.arange(F))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
            for p in parts:  # contiguous blocks
                assert len(p) == 0 or np.array_equal(p, np.arange(p[0], p[0] + len(p)))
    cost = np.array([10, 1, 1, 1, 1, 1, 1, 1, 1, 1], dtype=float)
    parts = [shard_frames(10, 2, r, cost=cost) for r in range(2)]
    loads = [cost[p].sum() for p in parts]
    assert sorted(np.concatenate(parts).tolist()) == list(range(10))
    assert max(loads) == 10.0 and min(loads) == 9.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2604_09643_b200 import gen
        from paper_2604_09643_b200._pa import make_allreduce_callback
        from paper_2604_09643_b200.dist import make_allreduce

        grid = gen.make_grid((6, 5, 4), 0.2)
        acq = gen.make_acq(200, 0.2, t0=1.0)
        tmpl = gen.linear_array(3, 0.3)
        e = np.zeros((5, 6))
        e[:, 4] = np.linspace(-0.4, 0.4, 5)
        e[:, 5] = grid["origin"][2] - 3.0
        poses = gen.poses_from_euler(e)
        cot = gen.random_cotangent((5, 3, 200), seed=3)
        fr = shard_frames(5, world, rank)
        z = torch.tensor(oracle.adjoint(grid, acq, tmpl, poses[fr], cot[fr]).ravel())
        loss = torch.tensor([0.0, float(len(fr))], dtype=torch.float64)
        cb = make_allreduce_callback([z, loss[1:2]], make_allreduce())
        rc1 = cb(z.data_ptr(), z.numel(), None, None)
        rc2 = cb(loss[1:2].data_ptr(), 1, None, None)
        rc3 = cb(12345, 1, None, None)  # unknown pointer -> failure code, no exception
        if rank == 0:
            full = oracle.adjoint(grid, acq, tmpl, poses, cot).ravel()
            q.put((rc1, rc2, rc3, float(np.max(np.abs(z.numpy() - full)) / np.max(np.abs(full))), float(loss[1])))
    finally:
        dist.destroy_process_group()


def test_allreduce_callback_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    rc1, rc2, rc3, err, nloss = q.get(timeout=10)
    assert rc1 == 0 and rc2 == 0 and rc3 != 0
    assert err <= 1e-12          # sum of the two shard adjoints == adjoint over all frames
    assert nloss == 5.0          # loss slot summed across ranks
