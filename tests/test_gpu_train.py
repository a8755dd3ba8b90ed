"""Device loss / SSIM gradient / Adam (csrc/train.cu) vs the reference's own
outputs (tests/golden/train, made by tests/golden/make_golden_train.py) and the
oracle restatement (oracle/train_oracle.py)."""
from pathlib import Path

import numpy as np
import pytest
import torch

from conftest import assert_close
from oracle import train_oracle as T

pytestmark = pytest.mark.gpu

TRAIN = Path(__file__).resolve().parent / "golden" / "train"
LOSS = sorted(TRAIN.glob("loss_*.npz"))
ADAM = sorted(TRAIN.glob("adam_*.npz"))


@pytest.mark.parametrize("path", LOSS, ids=[p.stem for p in LOSS])
def test_device_loss_matches_reference(path):
    from paper_2506_21633_b200 import train

    z = np.load(path)
    value, grad = train.loss(z["S"], z["Y"], float(z["lam"]), float(z["max_val"]))
    assert abs(value - float(z["value"])) <= 1e-12 * max(1.0, abs(float(z["value"]))), (value, float(z["value"]))
    assert_close(grad, z["grad"], atol=1e-15, rtol=1e-10, what="dL/dS")


def test_device_loss_stays_on_device_and_is_deterministic():
    from paper_2506_21633_b200 import train

    g = torch.Generator("cuda").manual_seed(2)
    S = torch.rand((96, 80), dtype=torch.float64, device="cuda", generator=g)
    Y = torch.rand((96, 80), dtype=torch.float64, device="cuda", generator=g)
    buf = train.LossBuffers(96, 80)
    v1, g1 = train.loss(S, Y, 0.2, 1.0, buffers=buf)
    v2, g2 = train.loss(S, Y, 0.2, 1.0, buffers=buf)
    assert v1.is_cuda and g1.is_cuda
    assert torch.equal(v1, v2) and torch.equal(g1, g2)
    ov, og = T.loss(S.cpu().numpy(), Y.cpu().numpy(), 0.2, 1.0)
    assert abs(float(v1) - ov) <= 1e-12
    assert_close(g1.cpu().numpy(), og, atol=1e-15, rtol=1e-10, what="dL/dS")


def _grads(z, k, n):
    from paper_2506_21633_b200.rasterizer import SceneGradients

    f = lambda g: torch.from_numpy(z[f"g{k}_{g}"].astype(np.float32)).cuda()  # noqa: E731
    return SceneGradients(f("positions"), f("rotations"), f("log_scales"), f("sh_coeffs"), f("ke_raw"),
                          torch.zeros(n, dtype=torch.float32, device="cuda"),
                          torch.ones(n, dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("path", ADAM, ids=[p.stem for p in ADAM])
def test_device_adam_fp64_matches_reference(path):
    from paper_2506_21633_b200 import train
    from paper_2506_21633_b200.scene import DeviceScene

    z = np.load(path)
    scene = DeviceScene(*(torch.from_numpy(z[f"p0_{g}"].copy()).cuda() for g in T.GROUPS))
    state = train.AdamState.for_scene(scene)
    lrs = dict(zip(T.GROUPS, z["lrs"]))
    bound = float(z["bound"])
    n = len(scene)
    for k in range(2):
        train.adam_step(scene, _grads(z, k, n), state, lrs, None if bound < 0 else bound)
        for g in T.GROUPS:
            assert_close(getattr(scene, g).cpu().numpy(), z[f"p{k + 1}_{g}"], atol=0.0, rtol=1e-15, what=g)
            assert_close(getattr(state.m, g).cpu().numpy(), z[f"m{k + 1}_{g}"], atol=0.0, rtol=1e-15, what=g)
            assert_close(getattr(state.v, g).cpu().numpy(), z[f"v{k + 1}_{g}"], atol=0.0, rtol=1e-15, what=g)
    assert state.n_skipped == int(z["n_skipped"])


def test_device_adam_fp32_scene_vs_oracle():
    from paper_2506_21633_b200 import train
    from paper_2506_21633_b200.scene import DeviceScene

    z = np.load(ADAM[0])
    p0 = {g: z[f"p0_{g}"].astype(np.float32).astype(np.float64) for g in T.GROUPS}
    scene = DeviceScene(*(torch.from_numpy(p0[g].astype(np.float32)).cuda() for g in T.GROUPS))
    state = train.AdamState.for_scene(scene)
    lrs = dict(zip(T.GROUPS, z["lrs"]))
    params = {g: p0[g].copy() for g in T.GROUPS}
    m = {g: np.zeros_like(params[g]) for g in T.GROUPS}
    v = {g: np.zeros_like(params[g]) for g in T.GROUPS}
    step = 0
    for k in range(2):
        train.adam_step(scene, _grads(z, k, len(scene)), state, lrs)
        step, _ = T.adam_step(params, {g: z[f"g{k}_{g}"] for g in T.GROUPS}, m, v, step, lrs)
        # the device keeps FP32 parameters and moments between steps
        for g in T.GROUPS:
            params[g] = params[g].astype(np.float32).astype(np.float64)
            m[g] = m[g].astype(np.float32).astype(np.float64)
            v[g] = v[g].astype(np.float32).astype(np.float64)
    for g in T.GROUPS:
        assert_close(getattr(scene, g).double().cpu().numpy(), params[g], atol=1e-6, rtol=1e-5, what=g)


def _toy_problem(n_views=3, size=64):
    import paper_2506_21633_b200 as sdgr
    from paper_2506_21633_b200 import targets
    from paper_2506_21633_b200.scene import DeviceScene

    tank = targets.to_float32_exact(targets.composite_target(targets.tank_preset(), [1500, 800, 300], seed=8))
    cfgs = [sdgr.RadarConfig(azimuth_deg=az, elevation_deg=45.0, altitude_m=0.5, n_range=size, n_azimuth=size)
            for az in np.linspace(0.0, 240.0, n_views)]
    truth = DeviceScene.from_host(tank, dtype=torch.float64)
    tg = torch.stack([torch.as_tensor(sdgr.render(truth, c)).cuda() for c in cfgs]).double()
    start = DeviceScene.from_host(tank, dtype=torch.float64)
    g = torch.Generator("cuda").manual_seed(1)
    start.positions += 0.05 * torch.randn(start.positions.shape, dtype=torch.float64, device="cuda", generator=g)
    return start, cfgs, tg


def test_trainstep_loss_and_dlds_match_standalone_loss():
    import paper_2506_21633_b200 as sdgr
    from paper_2506_21633_b200 import train

    scene, cfgs, tg = _toy_problem()
    ts = train.TrainStep(scene, cfgs, tg, lambda_ssim=0.2, geo_batch=2)
    ts.mv.run(ts.dlds, check=True)
    for i, c in enumerate(cfgs):
        img = torch.as_tensor(sdgr.render(scene, c)).cuda().double()
        v, gr = train.loss(img, tg[i], 0.2, 1.0)
        assert abs(float(ts.mv.loss_values[i]) - float(v)) <= 1e-10
        # the multi-view step cuts tile lists into longer depth segments than the
        # single-view render (multiview.MULTIVIEW_SEG_LEN), which re-associates
        # the fixed-point pass-A sums at the 1e-12 level; SSIM's gradient
        # amplifies that, so agreement is to 1e-6 relative, not bitwise
        assert_close(ts.dlds[i].cpu().numpy(), gr.cpu().numpy(), atol=1e-11, rtol=1e-6, what="dL/dS")


def test_trainstep_reduces_the_loss():
    from paper_2506_21633_b200 import train

    scene, cfgs, tg = _toy_problem()
    ts = train.TrainStep(scene, cfgs, tg, lambda_ssim=0.2, geo_batch=2)
    lrs = {"positions": 2e-3, "rotations": 1e-3, "log_scales": 5e-3, "sh_coeffs": 2.5e-3, "ke_raw": 5e-2}
    first = float(ts(lrs).sum())
    for _ in range(15):
        last = ts(lrs)
    ts.mv.check()
    assert float(last.sum()) < first
    assert ts.state.step == 16


def test_trainstep_overflow_recalibrates_and_reruns():
    """a step whose footprints outgrow the calibrated pair / replay
    capacity must not apply truncated gradients.  The device guard skips Adam,
    the step recalibrates (dropping the stale graph) and re-runs, and the
    update equals that of a step calibrated on the grown scene from the start."""
    from paper_2506_21633_b200 import train
    from paper_2506_21633_b200.scene import DeviceScene

    scene, cfgs, tg = _toy_problem()
    lrs = {"positions": 2e-3, "rotations": 1e-3, "log_scales": 5e-3, "sh_coeffs": 2.5e-3, "ke_raw": 5e-2}
    ts = train.TrainStep(scene, cfgs, tg, lambda_ssim=0.2, geo_batch=2, headroom=1.0)
    ts.mv.calibrate()                        # capacities of the original footprints
    ts.mv.capture(ts.dlds)                   # and a graph on those buffers
    ts.graph_generation = gen = ts.mv.generation
    scene.log_scales.add_(1.5)               # ~4.5x larger footprints than calibrated
    twin = DeviceScene(*(a.clone() for a in scene.arrays()))
    ts(lrs)                                  # overflows, recalibrates, re-runs
    assert ts.mv.generation > gen and ts.state.step == 1
    ref = train.TrainStep(twin, cfgs, tg, lambda_ssim=0.2, geo_batch=2)
    ref(lrs)
    for x, y in zip(scene.arrays(), twin.arrays()):
        assert torch.equal(x, y)
    with pytest.raises(OverflowError):       # without the check the guard still holds
        small = DeviceScene(*(a.clone() for a in twin.arrays()))
        t2 = train.TrainStep(small, cfgs, tg, lambda_ssim=0.2, geo_batch=2, headroom=1.0)
        t2.mv.calibrate()
        small.log_scales.add_(1.5)
        before = [a.clone() for a in small.arrays()]
        t2(lrs, check=False)
        assert all(torch.equal(x, y) for x, y in zip(small.arrays(), before))   # Adam skipped on device
        t2.mv.check()


def test_device_densify_matches_reference():
    from paper_2506_21633_b200 import densify, train
    from paper_2506_21633_b200.radar import RadarConfig
    from paper_2506_21633_b200.scene import DeviceScene

    z = np.load(TRAIN / "densify.npz")
    scene = DeviceScene(*(torch.from_numpy(z[f"in_{g}"].copy()).cuda() for g in T.GROUPS))
    state = train.AdamState.for_scene(scene)
    for g in T.GROUPS:
        getattr(state.m, g).copy_(torch.from_numpy(z[f"in_m_{g}"]))
        getattr(state.v, g).copy_(torch.from_numpy(z[f"in_v_{g}"]))
    acc = densify.GradAccumulator(torch.from_numpy(z["norm_sum"]).cuda(), torch.from_numpy(z["pos_sum"]).cuda(),
                                  torch.from_numpy(z["count"]).cuda())
    c = z["cfg"]
    cfg = densify.DensifyConfig(*map(float, c))
    view = RadarConfig(azimuth_deg=0.0, elevation_deg=45.0, range_res_m=0.3, n_range=64)
    assert abs(view.ground_extent_m - float(z["ground_extent"])) == 0.0
    out, acc2, ev = densify.densify_and_prune(scene, acc, cfg, view, float(z["extent"]), float(z["lr"]),
                                              np.random.default_rng(int(z["seed"])), state=state)
    assert (ev.n_cloned, ev.n_split, ev.n_pruned, ev.n_after) == tuple(int(x) for x in z["event"])
    for g in T.GROUPS:
        assert_close(getattr(out, g).cpu().numpy(), z[f"out_{g}"], atol=1e-14, rtol=1e-12, what=g)
        assert np.array_equal(getattr(state.m, g).cpu().numpy(), z[f"out_m_{g}"]), g
        assert np.array_equal(getattr(state.v, g).cpu().numpy(), z[f"out_v_{g}"]), g
    assert float(acc2.count.sum()) == 0.0 and acc2.count.shape[0] == ev.n_after


def test_device_accumulator_update():
    from paper_2506_21633_b200 import densify
    from paper_2506_21633_b200.rasterizer import SceneGradients

    n = 100
    g = torch.Generator("cuda").manual_seed(3)
    pos = torch.randn((n, 3), dtype=torch.float32, device="cuda", generator=g)
    uvn = torch.rand((n,), dtype=torch.float32, device="cuda", generator=g)
    vis = torch.randint(0, 3, (n,), dtype=torch.int32, device="cuda", generator=g)
    z = lambda *s: torch.zeros(s, dtype=torch.float32, device="cuda")  # noqa: E731
    grads = SceneGradients(pos, z(n, 4), z(n, 3), z(n, 16), z(n, 2), uvn, vis)
    acc = densify.GradAccumulator.zeros(n)
    acc.update(grads)
    acc.update(grads)
    m = (vis > 0).double()
    assert torch.equal(acc.count, 2 * vis.double())
    assert torch.allclose(acc.norm_sum, 2 * uvn.double() * m)
    assert torch.allclose(acc.pos_sum, 2 * pos.double() * m[:, None])
