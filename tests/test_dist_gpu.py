"""a7 on the real operator (-m gpu): two ranks on the one GPU of the test box, each running libpa's pa_step on
its frame shard with the all-reduce callback over a world-2 gloo process group (CUDA tensors), against a
single-rank pa_step over all frames (Stage 5 "coherently combining"; Alg. 1).

Nothing waits on a peer inside a kernel: the ranks meet only in the host-side gloo collective that pa_step
requests through its callback, so sharing one GPU is safe."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

F_ALL = 6


def _problem():
    import oracle
    from paper_2604_09643_b200 import gen

    grid = gen.make_grid((20, 18, 12), 0.2)
    grid = dict(grid, origin=[float(np.float32(o)) for o in grid["origin"]], pitch=float(np.float32(0.2)))
    acq = gen.make_acq(360, 0.2, t0=1.0)
    tmpl = gen.linear_array(10, 0.3)
    rng = np.random.default_rng(21)
    e_true = np.zeros((F_ALL, 6))
    e_true[:, :3] = rng.normal(scale=0.05, size=(F_ALL, 3))
    e_true[:, 3:5] = rng.normal(scale=0.4, size=(F_ALL, 2))
    e_true[:, 5] = -4.5 - rng.uniform(0, 0.5, size=F_ALL)
    p_true = gen.random_volume(grid, 22)
    meas = oracle.forward(grid, acq, tmpl, gen.poses_from_euler(e_true), p_true)
    e0 = e_true + rng.normal(scale=[0.01, 0.01, 0.01, 0.05, 0.05, 0.05], size=(F_ALL, 6))
    p0 = np.full(p_true.shape, 0.3)
    return grid, acq, tmpl, meas.astype(np.float32), p0.astype(np.float32), e0.astype(np.float32)


CFG = dict(lr_p0=1e-2, lr_rot=2e-3, lr_trans=1e-2, step=2, loss_kind=0)


def _run(ctx, frames, allreduce):
    from paper_2604_09643_b200 import Context  # noqa: F401

    grid, acq, tmpl, meas, p0, e0 = _problem()
    dev = torch.device("cuda", 0)
    nv = p0.size
    F = len(frames)
    p = torch.tensor(p0, device=dev)
    e = torch.tensor(e0[frames], device=dev)
    st_v = np.full(nv, 1e-6, dtype=np.float32)
    am = torch.cat([torch.zeros(nv, device=dev), torch.tensor(st_v, device=dev)])
    aq = torch.cat([torch.zeros(6 * F, device=dev), torch.full((6 * F,), 1e-4, device=dev)])
    g = torch.empty(nv, device=dev)
    L = torch.empty(2, device=dev)
    ctx.step(grid, acq, torch.tensor(tmpl, dtype=torch.float32, device=dev), torch.tensor(meas[frames], device=dev),
             p, e, am, aq, g, L, dict(CFG), allreduce=allreduce, check=True)
    torch.cuda.synchronize()
    return dict(grad=g.cpu().numpy(), p0=p.cpu().numpy(), euler=e.cpu().numpy(), loss=L.cpu().numpy())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_09643_b200 import Context
        from paper_2604_09643_b200.dist import make_allreduce, shard_frames

        ctx = Context(0)
        fr = shard_frames(F_ALL, world, rank)
        a = _run(ctx, fr, make_allreduce())
        b = _run(ctx, fr, make_allreduce())  # run-to-run: bitwise for a fixed world size
        q.put((rank, fr.tolist(), a, bool(all(np.array_equal(a[k], b[k]) for k in a))))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_equal_one_rank(record_parity):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    from paper_2604_09643_b200 import Context

    __graft_entry__.build()
    ref = _run(Context(0), np.arange(F_ALL), None)
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    res.sort(key=lambda r: r[0])
    rel = lambda a, b: float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))  # noqa: E731
    for rank, frames, out, bitwise in res:
        assert bitwise, rank
        # the all-reduced gradient, the replicated p0 update and the global loss equal the single-rank step
        record_parity(f"world2_rank{rank}_grad_p0", rel(out["grad"], ref["grad"]), 1e-6)
        assert rel(out["grad"], ref["grad"]) <= 1e-6
        assert rel(out["p0"].astype(np.float64) - 0.3, ref["p0"].astype(np.float64) - 0.3) <= 1e-5  # fp32 ulp(0.3) / update
        assert abs(out["loss"][1] - ref["loss"][0]) <= 1e-6 * abs(ref["loss"][0])
        # each rank's pose update is the single-rank update of its frames
        e0 = _problem()[5].astype(np.float64)[frames]
        assert rel(out["euler"] - e0, ref["euler"][frames] - e0) <= 1e-5
    # both ranks hold the identical p0 (replicated update)
    assert np.array_equal(res[0][2]["p0"], res[1][2]["p0"])
    assert np.array_equal(res[0][2]["grad"], res[1][2]["grad"])
