"""Multi-rank view sharding + gradient all-reduce on CPU (gloo, world size 2).

The device step (MultiViewStep) accumulates per-view gradients into one flat
SoA buffer and calls allreduce_grads once per step.  Here each rank fills the
same flat layout with the oracle's per-view gradients for its shard (a CPU
stand-in for the device step), runs the real allreduce_grads over gloo, and
the result must equal the oracle's sum over ALL views -- the multi-GPU parity
definition of SURVEY.md §8e.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GROUPS, assert_close


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene_and_views():
    from paper_2506_21633_b200 import targets
    from paper_2506_21633_b200.radar import RadarConfig

    scene = targets.random_scene(np.random.default_rng(5), 12)
    views = [RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=2.0, range_res_m=0.5, azimuth_res_m=0.5,
                         n_range=16, n_azimuth=16) for az in (10.0, 100.0, 190.0) for el in (40.0, 50.0)]
    return scene, views


def _oracle_grads(scene, cfg, seed):
    from oracle import sdgr_oracle as O
    f = O.render_forward(scene, cfg)
    return O.backward(f, np.random.default_rng(seed).normal(size=f.image.shape))


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_21633_b200.multiview import GRAD_WIDTH, allreduce_grads, grad_views, shard_views

    scene, views = _scene_and_views()
    n = len(scene)
    flat = torch.zeros(GRAD_WIDTH * n, dtype=torch.float32)
    g = grad_views(flat, n)
    idx = [i for i in range(len(views)) if i % world == rank]
    assert [views[i] for i in idx] == shard_views(views, rank, world)
    for i in idx:
        go = _oracle_grads(scene, views[i], i)
        for k in GROUPS + ("uv_grad_norm",):
            getattr(g, k).add_(torch.from_numpy(go[k].astype(np.float32)).reshape(getattr(g, k).shape))
        g.visible.add_(torch.from_numpy(go["visible"].astype(np.int32)))
    allreduce_grads(flat, n)
    if rank == 0:
        torch.save(flat, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_allreduce_equals_sum_over_views(tmp_path):
    out = tmp_path / "flat.pt"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    from paper_2506_21633_b200.multiview import grad_views

    scene, views = _scene_and_views()
    n = len(scene)
    got = grad_views(torch.load(out), n)
    ref = {k: 0 for k in GROUPS + ("uv_grad_norm", "visible")}
    for i, cfg in enumerate(views):
        go = _oracle_grads(scene, cfg, i)
        for k in ref:
            ref[k] = ref[k] + go[k].astype(np.float64)
    for k in GROUPS + ("uv_grad_norm",):
        a = getattr(got, k).numpy().astype(np.float64).reshape(ref[k].shape)
        assert_close(a, ref[k], what=k)   # north-star tolerance, FP32 storage
    assert np.array_equal(got.visible.numpy(), ref["visible"].astype(np.int32))


def _device_worker(rank, world, port, out_path):
    """One rank of a 2-rank view-sharded step on cuda:0: the real device step
    (MultiViewStep.run: batched preprocessing, walks, geometry epilogue) on
    this rank's shard, then its one all-reduce of the flat gradient buffer."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2506_21633_b200 as sdgr
    from paper_2506_21633_b200.multiview import MultiViewStep, shard_views

    tank, cfgs, dl = _device_problem()
    ds = sdgr.DeviceScene.from_host(tank, dtype=torch.float32)
    mine = shard_views(cfgs, rank, world)
    step = MultiViewStep(ds, mine)
    got = step.run(torch.from_numpy(dl[rank::world]).cuda())   # all-reduced inside run()
    if rank == 0:
        torch.save(step.flat_soa.cpu(), out_path)
    dist.barrier()
    dist.destroy_process_group()


def _device_problem():
    from paper_2506_21633_b200 import targets
    from paper_2506_21633_b200.radar import RadarConfig

    tank = targets.to_float32_exact(targets.composite_target(targets.tank_preset(), [3000, 1500, 500], seed=11))
    cfgs = [RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=0.5, n_range=96, n_azimuth=96)
            for az, el in ((0.0, 30.0), (70.0, 45.0), (140.0, 60.0), (210.0, 30.0), (280.0, 45.0))]
    dl = np.random.default_rng(17).normal(size=(len(cfgs), 96, 96))
    return tank, cfgs, dl


@pytest.mark.gpu
def test_two_rank_device_steps_allreduce_equals_oracle_sum(tmp_path):
    """SURVEY §8e multi-GPU parity on the hardware available: two ranks (gloo,
    both on cuda:0 -- their kernels never wait on each other; the exchange is
    the host-staged gloo all-reduce) each run MultiViewStep on their shard of
    five views; the all-reduced gradients equal the oracle's sum over all
    five views within the north-star tolerance, visible counts exactly."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    out = tmp_path / "flat.pt"
    mp.spawn(_device_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    from oracle import sdgr_oracle as O
    from paper_2506_21633_b200.multiview import grad_views

    tank, cfgs, dl = _device_problem()
    n = len(tank)
    got = grad_views(torch.load(out), n)
    ref = {k: 0.0 for k in GROUPS + ("uv_grad_norm", "visible")}
    for i, c in enumerate(cfgs):
        go = O.backward(O.render_forward(tank, c, exp="device"), dl[i])
        for k in ref:
            ref[k] = ref[k] + go[k].astype(np.float64)
    for k in GROUPS + ("uv_grad_norm",):
        assert_close(getattr(got, k).numpy().astype(np.float64).reshape(ref[k].shape), ref[k], what=k)
    assert np.array_equal(got.visible.numpy().astype(np.int64), ref["visible"].astype(np.int64))
