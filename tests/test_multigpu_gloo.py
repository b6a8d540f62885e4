"""Multi-rank (N > 1) host logic of batched mapping, on CPU with the gloo backend, world size 2
(the GPU box of this round has one GPU; the NCCL path is the same code with backend "nccl").

Checks: view sharding partitions the batch; the all-reduced 5N gradient buffer equals the
single-rank sum over all views (per-view gradients from the CPU oracle stand in for the per-rank
`vtgs_render_bwd` accumulation).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_02741_b200.mapping import GradBuffer, allreduce_grads, shard_views


@pytest.mark.parametrize("n_views", [1, 5, 8, 16])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_views_partition(n_views, world):
    shards = [shard_views(n_views, world, r) for r in range(world)]
    flat = [v for s in shards for v in s]
    assert flat == list(range(n_views))
    sizes = [len(s) for s in shards]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _views_and_grads():
    """4 views of one micro scene and each view's oracle gradient (d_col_opa | d_radius)."""
    import oracle
    from synth.scenes import micro_scene, perturb_pose
    m = micro_scene(7, n=40, width=24, height=20)
    rng = np.random.default_rng(0)
    views = [perturb_pose(m["view"], 3.0 * k, 0.01 * k, rng) for k in range(4)]
    grads = []
    H, W = m["intr"].height, m["intr"].width
    for k, v in enumerate(views):
        r = np.random.default_rng(100 + k)
        g = oracle.render_bwd(m["pos_rad"], m["col_opa"], v, m["intr"], r.normal(size=(H, W, 3)),
                              r.normal(size=(H, W)), r.normal(size=(H, W)), mode="f64")
        grads.append(np.concatenate([g["d_col_opa"].reshape(-1), g["d_radius"]]).astype(np.float32))
    return grads


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grads = _views_and_grads()
        n = grads[0].size // 5
        buf = GradBuffer(n, "cpu")
        for k in shard_views(len(grads), world, rank):          # this rank's views, accumulated (+=)
            buf.flat += torch.from_numpy(grads[k])
        allreduce_grads(buf)
        q.put((rank, buf.flat.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_allreduce_equals_single_rank_sum():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = np.sum(_views_and_grads(), axis=0, dtype=np.float64)
    for r in range(world):
        np.testing.assert_allclose(out[r], ref, rtol=1e-5, atol=1e-6)
    assert np.array_equal(out[0], out[1])   # identical buffers on every rank after the all-reduce


def _mapper_worker(rank, world, port, q):
    """One rank of BatchedMapper.step on config 1 with 4 views, gloo all-reduce of the CUDA
    gradient buffer (the NCCL path is the same call with backend "nccl")."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _mapper_step(rank, world)))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _mapper_step(rank, world):
    from paper_2506_02741_b200 import vtgs
    from paper_2506_02741_b200.mapping import BatchedMapper, shard_views
    from synth.scenes import make_config, perturb_pose
    cfg = make_config(1, 0)
    dev = "cuda"
    R = vtgs.Renderer(0, cfg.n_slots, cfg.intr.width, cfg.intr.height)
    pr, co = R.instantiate(torch.from_numpy(cfg.depth_stack()).to(dev), torch.from_numpy(cfg.rgb_stack()).to(dev),
                           vtgs.pose_tensor(cfg.pose_stack(), dev), cfg.intr, torch.from_numpy(cfg.opacity).to(dev))
    rng = np.random.default_rng(0)
    all_views = [perturb_pose(cfg.keyframes[0].pose, 1.0 * k, 0.01 * k, rng) for k in range(4)]
    mine = shard_views(len(all_views), world, rank)
    views = [vtgs.pose_tensor(np.asarray(all_views[k], dtype=np.float32), dev) for k in mine]
    tg = cfg.targets[0]
    tgts = [dict(rgb=torch.from_numpy(tg.rgb).to(dev), depth=torch.from_numpy(tg.depth).to(dev)) for _ in mine]
    m = BatchedMapper(R, pr, co, cfg.intr, views, tgts, 1.0, 0.5,
                      group=dist.group.WORLD if world > 1 else None)
    g = m.step(allreduce=False)            # this rank's views, accumulated
    torch.cuda.synchronize()
    local = g.flat.cpu().numpy().copy()
    if world > 1:
        from paper_2506_02741_b200.mapping import allreduce_grads
        allreduce_grads(g, m.group)
        torch.cuda.synchronize()
    return local, g.flat.cpu().numpy().copy()


@pytest.mark.gpu
def test_batched_mapper_two_ranks_equals_one():
    """BatchedMapper.step over 2 ranks (2 views each) with the all-reduce gives the same 5N
    gradient buffer on both ranks (exactly the sum of the two local buffers) as one rank
    rendering all 4 views (up to the float-atomic summation order)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mapper_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (l0, a0), (l1, a1) = out[0], out[1]
    # the all-reduce is exact plumbing: both ranks hold the fp32 sum of the two local buffers
    assert np.array_equal(a0, a1)
    assert np.array_equal(a0, l0 + l1)
    # and that sum is the single-rank gradient up to the float-atomic summation order, bounded by
    # the magnitudes of the two partial sums (a cancelling pair of partials rounds like its parts)
    _, ref = _mapper_step(0, 1)
    err = np.abs(a0.astype(np.float64) - ref)
    bound = 1e-4 * (np.abs(l0) + np.abs(l1) + np.abs(ref)) + 1e-6
    assert np.all(err <= bound), (err.max(), int(np.argmax(err - bound)))
