"""CUDA path vs the oracle and the reference's golden outputs (B200 only).

Bar (BASELINE.json north star): per-tile key lists and tile ranges
bit-exact; image, per-Gaussian intensity and every gradient column within
|gpu - ref| <= 1e-6 + 1e-4 |ref|.  Upstream gradients are O(1): N(0,1) and
dL/dS = S (gradcheck.py:79), per SURVEY.md §7 hard part 9.
"""
import math

import numpy as np
import pytest

from conftest import GROUPS, assert_close, npa, golden_files, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200 import targets  # noqa: E402
from paper_2506_21633_b200.rasterizer import decode_depth  # noqa: E402
from oracle import sdgr_oracle as O  # noqa: E402

GOLDEN = golden_files()


def tiles_np(tl):
    n = tl.n_pairs
    return (tl.pair_tile[:n].cpu().numpy().astype(np.int64), tl.tile_prim[:n].cpu().numpy().astype(np.int64),
            tl.tile_range.cpu().numpy().astype(np.int64))


def check_tiles(tl, ref_tile, ref_prim, ref_range, what):
    t, p, r = tiles_np(tl)
    assert t.shape == ref_tile.shape, (what, t.shape, ref_tile.shape)
    assert np.array_equal(t, ref_tile), what
    assert np.array_equal(p, ref_prim), what
    assert np.array_equal(r, ref_range), what


@pytest.mark.parametrize("path", GOLDEN, ids=[p.stem for p in GOLDEN])
@pytest.mark.parametrize("s_stop", [math.inf, sdgr.S_STOP], ids=["exact", "stop"])
def test_golden(path, s_stop):
    z, scene, cfg, cutoff = load_golden(path)
    fwd = sdgr.render_forward(scene, cfg, cutoff=cutoff, s_stop=s_stop)
    p = fwd.projection
    idx = npa(p.indices)
    assert np.array_equal(idx, z["indices"])
    assert p.n_culled == int(z["n_culled"]) and p.n_skipped == int(z["n_skipped"])
    # FP64 key chain: pixel centers and depth bit-identical to the reference
    assert np.array_equal(npa(p.uv_comp), z["uv_comp"])
    assert np.array_equal(npa(p.uv_img), z["uv_img"])
    assert np.array_equal(npa(p.depth), z["depth"])
    # covariances: exp(log-scale) is the only non-reference op (<= 1 ulp)
    assert_close(npa(p.cov_comp)[:, [0, 0, 1], [0, 1, 1]], z["cov_comp"], 1e-12, 1e-12, "cov_comp")
    assert_close(npa(p.cov_img)[:, [0, 0, 1], [0, 1, 1]], z["cov_img"], 1e-12, 1e-12, "cov_img")
    # bit-exact per-tile key lists and ranges, both planes
    check_tiles(fwd.rays, z["tiles0_tile"], z["tiles0_prim"], z["tiles0_range"], "comp tiles")
    check_tiles(fwd.splat, z["tiles1_tile"], z["tiles1_prim"], z["tiles1_range"], "img tiles")
    assert_close(npa(fwd.intensities.intensity), z["intensity"], what="intensity")
    assert_close(fwd.image.cpu().numpy() if hasattr(fwd.image, "cpu") else fwd.image, z["image"], what="image")
    rows = z["grad_rows"]
    for tag, dlds in (("n", z["dLdS"]), ("s", z["image"])):
        g = sdgr.backward(fwd, dlds)
        for k in GROUPS + ("uv_grad_norm",):
            assert_close(getattr(g, k)[rows], z[f"g{tag}_{k}"], what=f"{path.stem} grad {tag} {k}")
        assert np.array_equal(g.visible[rows], z[f"g{tag}_visible"])


def _oracle_compare(scene, cfg, cutoff, s_stop=sdgr.S_STOP, seed=0, device_scene=False):
    fo = O.render_forward(scene, cfg, cutoff=cutoff, exp="device")
    inp = sdgr.DeviceScene.from_host(scene, dtype=torch.float32) if device_scene else scene
    fwd = sdgr.render_forward(inp, cfg, cutoff=cutoff, s_stop=s_stop)
    img = fwd.image.cpu().numpy() if isinstance(fwd.image, torch.Tensor) else fwd.image
    assert_close(img, fo.image, what="image")
    for plane, pairs, tl in ((0, fo.rays, fwd.rays), (1, fo.spl, fwd.splat)):
        tt, gi, rg = O.tile_lists(pairs, fo.proj, plane)
        check_tiles(tl, tt, gi, rg, f"plane {plane}")
    # FP64 key chain bit-identical to the oracle's device-exp restatement
    p = fwd.projection
    assert np.array_equal(npa(p.cov_comp), fo.proj.cov_comp)
    assert np.array_equal(npa(p.depth), fo.proj.depth)
    rng = np.random.default_rng(seed)
    dlds = rng.normal(size=img.shape)
    go = O.backward(fo, dlds)
    g = sdgr.backward(fwd, torch.from_numpy(dlds).float().cuda() if device_scene else dlds)
    if device_scene:
        g = g.to_numpy()
    for k in GROUPS + ("uv_grad_norm",):
        assert_close(getattr(g, k), go[k], what=f"grad {k}")
    assert np.array_equal(g.visible, go["visible"])


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("cutoff", [math.inf, 3.0], ids=["dense", "cut"])
def test_random_small_vs_oracle(seed, cutoff):
    rng = np.random.default_rng(100 + seed)
    scene = targets.random_scene(rng, 4 + 3 * seed)
    cfg = sdgr.RadarConfig(azimuth_deg=float(rng.uniform(0, 360)), elevation_deg=float(rng.uniform(38, 52)),
                           altitude_m=float(rng.uniform(1, 4)), range_res_m=0.5, azimuth_res_m=0.5,
                           n_range=16 + 8 * (seed % 3), n_azimuth=16 + 5 * (seed % 2))
    _oracle_compare(scene, cfg, cutoff, seed=seed)


def test_float32_device_scene_matches_oracle():
    tank = targets.to_float32_exact(targets.composite_target(targets.tank_preset(), [3000, 1500, 500], seed=4))
    cfg = sdgr.RadarConfig(azimuth_deg=10.0, elevation_deg=50.0, altitude_m=0.5, n_range=128, n_azimuth=128)
    _oracle_compare(tank, cfg, 3.0, device_scene=True)


@pytest.mark.parametrize("el", [15.0, 45.0, 75.0])
def test_c2_tank_100k_vs_oracle(el):
    tank = targets.composite_target(targets.tank_preset(), [60000, 30000, 10000], seed=3)
    cfg = sdgr.RadarConfig(azimuth_deg=30.0, elevation_deg=el, altitude_m=0.5, n_range=256, n_azimuth=256)
    _oracle_compare(tank, cfg, 3.0, seed=int(el))


def test_perturbed_large_gaussians_vs_oracle():
    # footprints wider than the 8x8 cell window exercise the exact FP64 fallback
    rng = np.random.default_rng(9)
    scene = targets.random_scene(rng, 300, spread=6.0, scale_low=0.3, scale_high=2.0)
    cfg = sdgr.RadarConfig(azimuth_deg=33.0, elevation_deg=40.0, altitude_m=1.0, range_res_m=0.25,
                           azimuth_res_m=0.25, n_range=64, n_azimuth=80)
    _oracle_compare(scene, cfg, 3.0, seed=3)


def test_depth_key_roundtrip():
    d = torch.tensor([-3.5, -0.0, 0.0, 1e-300, 2.0, -1e-300, 7.25], dtype=torch.float64)
    from paper_2506_21633_b200.rasterizer import decode_depth as dec
    b = d.view(torch.int64)
    sign = b < 0
    key = torch.where(sign, ~b, b ^ torch.tensor(-0x8000000000000000, dtype=torch.int64))
    out = dec(key)
    assert torch.equal(out.abs(), d.abs())


def test_depth_order_api_matches_lexsort():
    """sdgr_depth_order (kept as a standalone C-ABI utility; the binning no
    longer needs a global order): visible Gaussians by (depth, index)."""
    import ctypes as C

    from paper_2506_21633_b200 import _lib

    tank = targets.composite_target(targets.tank_preset(), [4000, 2000, 1000], seed=9)
    cfg = sdgr.RadarConfig(azimuth_deg=33.0, elevation_deg=50.0, altitude_m=0.5, n_range=96, n_azimuth=96)
    proj = sdgr.project_all(tank, cfg)
    n = proj.n_scene
    lib = _lib.lib()
    ws_bytes = lib.sdgr_workspace_bytes(n, 1)
    ws = torch.empty((ws_bytes,), dtype=torch.uint8, device="cuda")
    order = torch.empty((n,), dtype=torch.int32, device="cuda")
    assert lib.sdgr_depth_order(C.byref(proj.desc()), order.data_ptr(), ws.data_ptr(), ws_bytes, None) == 0
    torch.cuda.synchronize()
    vis = ((proj.flags & _lib.FLAG_VISIBLE) != 0).cpu().numpy()
    depth = decode_depth(proj.depth_key).cpu().numpy()
    idx = np.nonzero(vis)[0]
    want = idx[np.lexsort((idx, depth[idx]))]
    assert np.array_equal(order.cpu().numpy()[: idx.size], want)


def test_empty_and_culled():
    cfg = sdgr.RadarConfig(azimuth_deg=20.0, elevation_deg=40.0, altitude_m=2.0, range_res_m=0.5,
                           azimuth_res_m=0.5, n_range=16, n_azimuth=16)
    img = sdgr.render(sdgr.Scene.empty(), cfg)
    assert img.shape == (16, 16) and np.all(img == 0)
    with pytest.raises(sdgr.NumericalError):
        sdgr.render_forward(sdgr.Scene.empty(), cfg)
    with pytest.raises(sdgr.InvalidParameterError):
        sdgr.project_all(sdgr.Scene.empty(), cfg)
    far = targets.random_scene(np.random.default_rng(0), 3)
    far.positions[:] = 100.0
    fwd = sdgr.render_forward(far, cfg)
    assert np.all(fwd.image == 0)
    g = sdgr.backward(fwd, np.ones((16, 16)))
    assert not g.visible.any() and np.all(g.positions == 0)


def test_nonfinite_names_primitive():
    cfg = sdgr.RadarConfig(azimuth_deg=20.0, elevation_deg=40.0, altitude_m=2.0, range_res_m=0.5,
                           azimuth_res_m=0.5, n_range=16, n_azimuth=16)
    scene = targets.random_scene(np.random.default_rng(3), 6)
    scene.sh_coeffs[4, 0] = np.inf
    with pytest.raises(sdgr.NumericalError, match="primitive 4"):
        sdgr.render_forward(scene, cfg)


def test_backward_state_errors():
    cfg = sdgr.RadarConfig(azimuth_deg=20.0, elevation_deg=40.0, altitude_m=2.0, range_res_m=0.5,
                           azimuth_res_m=0.5, n_range=16, n_azimuth=16)
    scene = targets.random_scene(np.random.default_rng(4), 4)
    fwd = sdgr.render_forward(scene, cfg)
    with pytest.raises(sdgr.StateError):
        sdgr.backward(fwd, np.zeros((3, 3)))
    bad = np.zeros((16, 16))
    bad[0, 0] = np.nan
    with pytest.raises(sdgr.InvalidParameterError):
        sdgr.backward(fwd, bad)
    scene.positions = np.vstack([scene.positions, np.zeros((1, 3))])
    with pytest.raises(sdgr.StateError):
        sdgr.backward(fwd, np.zeros((16, 16)))


def test_linearity_and_zero_gradient():
    cfg = sdgr.RadarConfig(azimuth_deg=20.0, elevation_deg=40.0, altitude_m=2.0, range_res_m=0.5,
                           azimuth_res_m=0.5, n_range=16, n_azimuth=16)
    rng = np.random.default_rng(5)
    scene = targets.random_scene(rng, 6)
    fwd = sdgr.render_forward(scene, cfg)
    z = sdgr.backward(fwd, np.zeros((16, 16)))
    for a in z.param_arrays():
        assert np.all(a == 0)
    g1, g2 = rng.normal(size=(16, 16)), rng.normal(size=(16, 16))
    lhs = sdgr.backward(fwd, 0.7 * g1 - 1.3 * g2)
    r1, r2 = sdgr.backward(fwd, g1), sdgr.backward(fwd, g2)
    for k in GROUPS:
        assert_close(getattr(lhs, k), 0.7 * getattr(r1, k) - 1.3 * getattr(r2, k), atol=1e-5, what=k)


@pytest.mark.parametrize("cutoff", [math.inf, 3.0], ids=["dense", "cut"])
def test_replay_equals_rewalk(cutoff):
    """The backward replaying the forward's live-pair log must give the same
    gradients as re-walking the tile lists (both deterministic)."""
    rng = np.random.default_rng(21)
    scene = targets.random_scene(rng, 40, spread=3.0)
    cfg = sdgr.RadarConfig(azimuth_deg=60.0, elevation_deg=45.0, altitude_m=2.0, range_res_m=0.25,
                           azimuth_res_m=0.25, n_range=48, n_azimuth=40)
    fwd = sdgr.render_forward(scene, cfg, cutoff=cutoff)
    g = rng.normal(size=(48, 40))
    a = sdgr.backward(fwd, g, use_replay=True)
    b = sdgr.backward(fwd, g, use_replay=False)
    for k in GROUPS + ("uv_grad_norm",):
        assert_close(getattr(a, k), getattr(b, k), atol=1e-12, rtol=1e-10, what=k)


def test_bitwise_determinism():
    tank = targets.composite_target(targets.tank_preset(), [6000, 3000, 1000], seed=5)
    cfg = sdgr.RadarConfig(azimuth_deg=77.0, elevation_deg=40.0, altitude_m=0.5, n_range=128, n_azimuth=128)
    g = np.random.default_rng(0).normal(size=(128, 128))
    outs = []
    for _ in range(2):
        fwd = sdgr.render_forward(tank, cfg)
        outs.append((fwd.image.copy(), sdgr.backward(fwd, g)))
    assert np.array_equal(outs[0][0], outs[1][0])
    for k in GROUPS + ("uv_grad_norm",):
        assert np.array_equal(getattr(outs[0][1], k), getattr(outs[1][1], k)), k


def oracle_sum(scene, cfgs, dl, cutoff=3.0):
    """Sum over views of the oracle's gradients (FP64) and visible counts:
    the multi-view parity definition of SURVEY.md §8e."""
    ref = {k: 0.0 for k in GROUPS + ("uv_grad_norm",)}
    vis = 0
    for i, c in enumerate(cfgs):
        fo = O.render_forward(scene, c, cutoff=cutoff, exp="device")
        go = O.backward(fo, dl[i].cpu().numpy())
        for k in ref:
            ref[k] = ref[k] + go[k]
        vis = vis + go["visible"].astype(np.int64)
    return ref, vis


def check_step_vs_oracle(got, ref, vis):
    for k in ref:
        assert_close(getattr(got, k).double().cpu().numpy(), ref[k], what=k)   # north-star tolerance
    assert np.array_equal(got.visible.cpu().numpy().astype(np.int64), vis)


@pytest.mark.parametrize("geo_batch", [1, 2, 8])
def test_multiview_step_equals_sum_of_views(geo_batch):
    """Batched geometry epilogue (1, partial and full batches) == the oracle's
    sum of single-view backward passes."""
    from paper_2506_21633_b200.multiview import MultiViewStep

    tank = targets.to_float32_exact(targets.composite_target(targets.tank_preset(), [3000, 1500, 500], seed=6))
    cfgs = [sdgr.RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=0.5, n_range=96, n_azimuth=96)
            for az, el in ((0.0, 30.0), (90.0, 45.0), (200.0, 60.0))]
    ds = sdgr.DeviceScene.from_host(tank, dtype=torch.float32)
    step = MultiViewStep(ds, cfgs, geo_batch=geo_batch)
    dl = torch.randn((3, 96, 96), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    got = step.run(dl)
    check_step_vs_oracle(got, *oracle_sum(tank, cfgs, dl))


def test_multiview_batch_ramp_vs_oracle():
    """A step whose batches ramp up (2, 6, 2 views with 8-view batches: three
    batches over both slot sets) equals the oracle's sum over its views."""
    from paper_2506_21633_b200.multiview import MultiViewStep

    tank = targets.to_float32_exact(targets.composite_target(targets.tank_preset(), [2000, 1000, 500], seed=7))
    cfgs = [sdgr.RadarConfig(azimuth_deg=float(az), elevation_deg=el, altitude_m=0.5, n_range=80, n_azimuth=80)
            for az, el in zip(range(0, 360, 36), (30.0, 45.0, 60.0) * 4)]
    ds = sdgr.DeviceScene.from_host(tank, dtype=torch.float32)
    step = MultiViewStep(ds, cfgs, geo_batch=8, ramp=2)
    assert step.batches == [2, 6, 2]
    dl = torch.randn((len(cfgs), 80, 80), dtype=torch.float64, device="cuda",
                     generator=torch.Generator("cuda").manual_seed(8))
    got = step.run(dl)
    check_step_vs_oracle(got, *oracle_sum(tank, cfgs, dl))


def test_multiview_graph_replay_equals_run():
    """The captured CUDA graph of a step reproduces run() bitwise, and reads
    its static inputs in place (new dL/dS values are picked up on replay)."""
    from paper_2506_21633_b200.multiview import MultiViewStep

    tank = targets.to_float32_exact(targets.composite_target(targets.tank_preset(), [3000, 1500, 500], seed=4))
    cfgs = [sdgr.RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=0.5, n_range=96, n_azimuth=96)
            for az, el in ((10.0, 30.0), (130.0, 60.0), (250.0, 45.0))]
    ds = sdgr.DeviceScene.from_host(tank, dtype=torch.float32)
    step = MultiViewStep(ds, cfgs, geo_batch=2)
    gen = torch.Generator("cuda").manual_seed(5)
    dl = torch.randn((3, 96, 96), dtype=torch.float64, device="cuda", generator=gen)
    step.run(dl)
    want = step.flat_soa.clone()
    assert step.capture(dl) > 0
    step.graph_step(check=True)
    assert torch.equal(step.flat_soa, want)
    dl.copy_(torch.randn((3, 96, 96), dtype=torch.float64, device="cuda", generator=gen))
    step.run(dl)
    want2 = step.flat_soa.clone()
    step.graph_step(check=True)
    assert torch.equal(step.flat_soa, want2)


def test_host_pipeline_equals_run():
    """HostStepPipeline (two banks, overlapped H2D / D2H) returns, for each
    submitted step, exactly run()'s gradients for that step's host inputs."""
    from paper_2506_21633_b200.multiview import HostStepPipeline, MultiViewStep

    tank = targets.to_float32_exact(targets.composite_target(targets.tank_preset(), [3000, 1500, 500], seed=4))
    cfgs = [sdgr.RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=0.5, n_range=96, n_azimuth=96)
            for az, el in ((10.0, 30.0), (130.0, 60.0), (250.0, 45.0))]
    ds = sdgr.DeviceScene.from_host(tank, dtype=torch.float32)
    step = MultiViewStep(ds, cfgs, geo_batch=2)
    pipe = HostStepPipeline(step, dl_dtype=torch.float32)
    g = torch.Generator().manual_seed(3)
    groups = ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")
    inputs, outs, wants = [], [], []
    for k in range(4):   # perturbed scenes so every step's result differs
        sc = {nm: (getattr(ds, nm).cpu() + (1e-3 * k if nm == "positions" else 0.0)).pin_memory() for nm in groups}
        dl = torch.randn((3, 96, 96), generator=g, dtype=torch.float32).pin_memory()
        inputs.append((sc, dl))
        outs.append(torch.empty(step.flat_soa.shape, dtype=torch.float32).pin_memory())
    for k, (sc, dl) in enumerate(inputs):
        pipe.submit(sc, dl, outs[k])
    pipe.drain()
    torch.cuda.synchronize()
    pipe.check()
    for k, (sc, dl) in enumerate(inputs):
        for nm in groups:
            getattr(ds, nm).copy_(sc[nm])
        step.run(dl.cuda().double())
        assert torch.equal(outs[k], step.flat_soa.cpu()), k


def test_multiview_capacity_overflow_is_detected():
    """Pair buffers are sized by calibration; a scene that later needs more
    pairs (grown footprints) must raise OverflowError from check(), never
    write past the buffers, and recalibration must recover the exact result."""
    from paper_2506_21633_b200.multiview import MultiViewStep

    tank = targets.to_float32_exact(targets.composite_target(targets.tank_preset(), [3000, 1500, 500], seed=4))
    cfgs = [sdgr.RadarConfig(azimuth_deg=az, elevation_deg=45.0, altitude_m=0.5, n_range=96, n_azimuth=96)
            for az in (10.0, 130.0)]
    ds = sdgr.DeviceScene.from_host(tank, dtype=torch.float32)
    step = MultiViewStep(ds, cfgs, geo_batch=2, headroom=1.0)
    dl = torch.randn((2, 96, 96), dtype=torch.float64, device="cuda",
                     generator=torch.Generator("cuda").manual_seed(2))
    step.run(dl)
    ds.log_scales.add_(1.5)          # ~4.5x larger footprints: far more pairs than calibrated
    with pytest.raises(OverflowError):
        step.run(dl)
    torch.cuda.synchronize()         # no illegal address
    step.calibrate()
    got = step.run(dl)
    ref = MultiViewStep(ds, cfgs, geo_batch=2).run(dl)
    assert torch.equal(got.positions, ref.positions) and torch.equal(got.visible, ref.visible)
    assert step.graph is None   # calibrate() dropped any graph captured on the old buffers


def test_depth_ties_and_near_ties_vs_oracle():
    """Exact (depth, index) order with duplicated positions (ties -> index
    order) and positions 1e-12 m apart (runs of equal 32-bit depth keys)."""
    rng = np.random.default_rng(31)
    base = targets.random_scene(rng, 300, spread=2.0, scale_low=0.2, scale_high=0.5)
    reps = [base]
    for eps in (0.0, 1e-12, -3e-12):
        s = base.copy()
        s.positions = s.positions + eps
        reps.append(s)
    scene = targets.concatenate(reps)
    perm = rng.permutation(len(scene))
    scene = sdgr.Scene(*(getattr(scene, g)[perm] for g in GROUPS))
    cfg = sdgr.RadarConfig(azimuth_deg=15.0, elevation_deg=45.0, altitude_m=2.0, range_res_m=0.25,
                           azimuth_res_m=0.25, n_range=48, n_azimuth=48)
    _oracle_compare(scene, cfg, 3.0, seed=31)


@pytest.mark.parametrize("n_views", [1, 3, 8, 16])
def test_batched_preprocessing_equals_single_views(n_views):
    """sdgr_project_batch + sdgr_depth_order_batch + sdgr_bin_batch (one launch
    per stage over the batch, packed / emit rows, fused count + emit) produce
    bit-identical per-tile key lists, tile ranges, packed pair records and
    work items to the single-view entry points, view by view."""
    from paper_2506_21633_b200.multiview import MultiViewStep

    tank = targets.to_float32_exact(targets.composite_target(targets.tank_preset(), [6000, 3000, 1000], seed=8))
    angles = [(az, el) for el in (30.0, 45.0, 60.0) for az in (0.0, 50.0, 130.0, 200.0, 290.0, 340.0)][:n_views]
    cfgs = [sdgr.RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=0.5, n_range=128, n_azimuth=128)
            for az, el in angles]
    ds = sdgr.DeviceScene.from_host(tank, dtype=torch.float32)
    step = MultiViewStep(ds, cfgs)
    step.calibrate()
    step._preprocess(step.views, 0)
    torch.cuda.synchronize()
    for k, c in enumerate(cfgs):
        fwd = sdgr.render_forward(ds, c)
        tl = fwd.rays
        n = tl.n_pairs
        t = step.slot_t[k]
        assert int(step.slot_offsets[k][step.n].item()) == n, f"view {k}: pair count"
        assert torch.equal(t["pair_tile"][:n].cpu(), tl.pair_tile[:n].cpu()), f"view {k}: tiles"
        assert torch.equal(t["pair_prim"][:n].cpu(), tl.tile_prim[:n].cpu()), f"view {k}: key lists"
        assert torch.equal(t["tile_range"].cpu(), tl.tile_range.cpu()), f"view {k}: tile ranges"
        assert torch.equal(t["pair_start"].cpu(), tl.pair_start.cpu()), f"view {k}: pair starts"
        assert torch.equal(t["pair_rec"][:n].cpu(), tl.pair_rec[:n].cpu()), f"view {k}: pair records"
        assert int(t["n_items"][1].item()) == 0, f"view {k}: overflow"
        if step.slot_tiles[k].seg_len == tl.seg_len:   # segment length follows the pair capacity
            ni = int(t["n_items"][0].item())
            assert ni == int(tl.n_items[0].item())
            assert torch.equal(t["items"][:ni].cpu(), tl.items[:ni].cpu()), f"view {k}: work items"


@pytest.mark.parametrize("cutoff", [3.0, math.inf], ids=["cut", "dense"])
def test_batched_preprocessing_small_scenes(cutoff):
    """Batched vs single-view binning on gradcheck-sized scenes, including the
    dense all-pairs mode (cutoff = inf, reference forward.py:80-84) and
    Gaussians larger than the 8x8 windows (exact re-enumeration paths)."""
    from paper_2506_21633_b200.multiview import MultiViewStep

    rng = np.random.default_rng(4)
    n = 300
    host = sdgr.Scene(positions=rng.uniform(-4, 4, size=(n, 3)),
                      rotations=rng.normal(size=(n, 4)),
                      log_scales=rng.uniform(np.log(0.05), np.log(2.5), size=(n, 3)),
                      sh_coeffs=np.column_stack([rng.uniform(1, 3, n), rng.normal(0, 0.1, (n, 15))]),
                      ke_raw=rng.uniform(-0.5, 1.0, size=(n, 2)))
    host = targets.to_float32_exact(host)
    cfgs = [sdgr.RadarConfig(azimuth_deg=az, elevation_deg=45.0, altitude_m=0.5, n_range=40, n_azimuth=40)
            for az in (0.0, 70.0, 140.0, 250.0)]
    ds = sdgr.DeviceScene.from_host(host, dtype=torch.float32)
    step = MultiViewStep(ds, cfgs, geo_batch=4, cutoff=cutoff)
    step.calibrate()
    step._preprocess(step.views, 0)
    torch.cuda.synchronize()
    for k, c in enumerate(cfgs):
        tl = sdgr.render_forward(ds, c, cutoff=cutoff).rays
        m = tl.n_pairs
        t = step.slot_t[k]
        assert int(step.slot_offsets[k][step.n].item()) == m
        assert torch.equal(t["pair_prim"][:m].cpu(), tl.tile_prim[:m].cpu()), f"view {k}: key lists"
        assert torch.equal(t["tile_range"].cpu(), tl.tile_range.cpu()), f"view {k}: tile ranges"
        assert torch.equal(t["pair_rec"][:m].cpu(), tl.pair_rec[:m].cpu()), f"view {k}: pair records"


def test_multiview_batch_with_a_view_that_sees_nothing():
    """A batch where one view culls every Gaussian (zero pairs: empty sort,
    empty tile lists, no work items) next to normal views: the step still
    equals the sum of the single-view passes, and the empty view adds nothing."""
    from paper_2506_21633_b200.multiview import MultiViewStep

    tank = targets.composite_target(targets.tank_preset(), [2000, 1000, 500], seed=2)
    tank.positions[:, 0] += 30.0                          # the target sits 30 m off the scene origin
    tank = targets.to_float32_exact(tank)
    wide = dict(range_res_m=1.5, azimuth_res_m=1.5, n_range=96, n_azimuth=96)     # 144 m frames: see it
    narrow = dict(range_res_m=0.2, azimuth_res_m=0.2, n_range=96, n_azimuth=96)   # 19 m frame: culls all
    cfgs = [sdgr.RadarConfig(azimuth_deg=30.0, elevation_deg=45.0, altitude_m=0.5, **wide),
            sdgr.RadarConfig(azimuth_deg=0.0, elevation_deg=45.0, altitude_m=0.5, **narrow),
            sdgr.RadarConfig(azimuth_deg=250.0, elevation_deg=60.0, altitude_m=0.5, **wide)]
    ds = sdgr.DeviceScene.from_host(tank, dtype=torch.float32)
    empty = sdgr.render_forward(ds, cfgs[1])
    assert empty.rays.n_pairs == 0 and not bool(empty.projection.visible.any())
    step = MultiViewStep(ds, cfgs)
    dl = torch.randn((3, 96, 96), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    got = step.run(dl)
    check_step_vs_oracle(got, *oracle_sum(tank, cfgs, dl))


def test_multiview_rejects_mixed_ray_grids():
    """Slot buffers are sized from the first view: a step whose views differ
    in the computation-plane grid (ray_grid) is refused up front."""
    from paper_2506_21633_b200.multiview import MultiViewStep

    tank = targets.composite_target(targets.tank_preset(), [300, 150, 50], seed=2)
    ds = sdgr.DeviceScene.from_host(tank, dtype=torch.float32)
    cfgs = [sdgr.RadarConfig(azimuth_deg=0.0, elevation_deg=45.0, altitude_m=0.5, n_range=64, n_azimuth=64),
            sdgr.RadarConfig(azimuth_deg=90.0, elevation_deg=45.0, altitude_m=0.5, n_range=64, n_azimuth=64,
                             ray_grid=(96, 80))]
    with pytest.raises(ValueError, match="ray grid"):
        MultiViewStep(ds, cfgs)


def test_host_callers_get_float64_gradients():
    """render_forward(host scene) + backward return FP64 numpy gradients, like
    the reference (backward.py:25-50); device callers get float32 tensors."""
    scene = targets.random_scene(np.random.default_rng(8), 20)
    cfg = sdgr.RadarConfig(azimuth_deg=20.0, elevation_deg=40.0, altitude_m=2.0, range_res_m=0.5,
                           azimuth_res_m=0.5, n_range=24, n_azimuth=24)
    g = sdgr.backward(sdgr.render_forward(scene, cfg), np.ones((24, 24)))
    assert all(a.dtype == np.float64 for a in g.param_arrays()) and g.visible.dtype == bool
    fo = O.render_forward(scene, cfg, exp="device")
    go = O.backward(fo, np.ones((24, 24)))
    for k in GROUPS:   # FP64 all the way: far inside the north-star tolerance
        assert_close(getattr(g, k), go[k], atol=1e-12, rtol=1e-9, what=k)
    ds = sdgr.DeviceScene.from_host(scene, dtype=torch.float32)
    gd = sdgr.backward(sdgr.render_forward(ds, cfg), torch.ones((24, 24), device="cuda"))
    assert gd.positions.dtype == torch.float32 and gd.positions.is_cuda


@pytest.mark.parametrize("case", ["equal_depths", "depth_outlier"])
def test_depth_order_long_runs(case):
    """runs of equal 24-bit depth keys longer than k_fix_runs'
    per-thread window (many Gaussians at one depth, or one far outlier along
    the line of sight squeezing every other depth into a few buckets) are
    sorted by the block-serial radix pass -- exact (depth, index) order, and
    the full pipeline still matches the oracle."""
    import ctypes as C

    from paper_2506_21633_b200 import _lib
    from paper_2506_21633_b200.radar import radar_rotation

    rng = np.random.default_rng(41)
    base = targets.random_scene(rng, 400, spread=2.0, scale_low=0.2, scale_high=0.5)
    cfg = sdgr.RadarConfig(azimuth_deg=25.0, elevation_deg=45.0, altitude_m=2.0, range_res_m=0.25,
                           azimuth_res_m=0.25, n_range=48, n_azimuth=48)
    R = radar_rotation(cfg.azimuth_deg, cfg.elevation_deg)
    if case == "equal_depths":
        # 300 Gaussians share one depth: spread only across the radar's x / y axes
        t = rng.uniform(-2, 2, size=(300, 2))
        base.positions[:300] = base.positions[0] + t[:, :1] * R[0] + t[:, 1:] * R[1]
    else:
        base.positions[7] = base.positions[7] + 1.0e5 * R[2]   # same pixel, 100 km deeper
    proj = sdgr.project_all(base, cfg)
    n = proj.n_scene
    lib = _lib.lib()
    ws_bytes = lib.sdgr_workspace_bytes(n, 1)
    ws = torch.empty((ws_bytes,), dtype=torch.uint8, device="cuda")
    order = torch.empty((n,), dtype=torch.int32, device="cuda")
    assert lib.sdgr_depth_order(C.byref(proj.desc()), order.data_ptr(), ws.data_ptr(), ws_bytes, None) == 0
    vis = ((proj.flags & _lib.FLAG_VISIBLE) != 0).cpu().numpy()
    depth = decode_depth(proj.depth_key).cpu().numpy()
    idx = np.nonzero(vis)[0]
    want = idx[np.lexsort((idx, depth[idx]))]
    assert np.array_equal(order.cpu().numpy()[: idx.size], want)
    _oracle_compare(base, cfg, 3.0, seed=41)


def test_registered_scene_arrays_track_in_place_updates():
    """The drop-in path page-locks scene arrays it sees again (scene.upload_f64):
    the uploads then DMA from the caller's own memory, so an in-place update
    between calls (the reference's adam_step, optimize.py:206) must be what the
    next call renders -- identical to rendering a fresh copy (staging path)."""
    import gc

    from paper_2506_21633_b200 import scene as scene_mod

    tank = targets.composite_target(targets.tank_preset(), [30000, 8000, 2000], seed=3)
    cfg = sdgr.RadarConfig(azimuth_deg=31.0, elevation_deg=45.0, altitude_m=0.5, n_range=128, n_azimuth=128)
    g = np.random.default_rng(1).normal(size=(128, 128))
    rng = np.random.default_rng(2)
    for call in range(4):
        fwd = sdgr.render_forward(tank, cfg)
        got = (fwd.image.copy(), sdgr.backward(fwd, g))
        fresh = sdgr.Scene(*(np.array(getattr(tank, k), copy=True) for k in GROUPS))
        fwd2 = sdgr.render_forward(fresh, cfg)
        ref = (fwd2.image.copy(), sdgr.backward(fwd2, g))
        assert np.array_equal(got[0], ref[0]), call
        for k in GROUPS + ("uv_grad_norm",):
            assert np.array_equal(getattr(got[1], k), getattr(ref[1], k)), (call, k)
        tank.positions += rng.normal(scale=1e-3, size=tank.positions.shape)   # in place
        tank.sh_coeffs *= 1.01
    big = [getattr(tank, k) for k in GROUPS if getattr(tank, k).nbytes >= scene_mod._REGISTER_MIN]
    def owner(a):
        while isinstance(a.base, np.ndarray):
            a = a.base
        return a

    states = {e[3] for e in scene_mod._SEEN.values() if any(e[0]() is owner(a) for a in big)}
    assert states == {"pinned"}, states
    n_seen = len(scene_mod._SEEN)
    del tank, fwd, fresh, fwd2, big
    gc.collect()
    assert len(scene_mod._SEEN) < n_seen


def test_result_blocks_recycle_only_when_unreferenced():
    """download() hands out numpy views of recycled page-locked blocks: a block
    holding any live array (or any view of one) is never written again."""
    import gc

    from paper_2506_21633_b200 import scene as scene_mod

    dev = torch.device("cuda", 0)
    a = torch.arange(300000, dtype=torch.float64, device=dev).reshape(-1, 3)
    b = torch.arange(100000, dtype=torch.float32, device=dev)
    r1 = scene_mod.download([a, b])
    assert np.array_equal(r1[0], npa(a)) and np.array_equal(r1[1], npa(b))
    keep = r1[0][:, 1]                       # a view of a view keeps block 1 alive
    del r1
    gc.collect()
    r2 = scene_mod.download([a * 2, b * 2])
    assert np.array_equal(keep, npa(a)[:, 1])   # untouched
    assert np.array_equal(r2[0], npa(a) * 2)
    blk2 = r2[0].base
    del keep, r2
    gc.collect()
    r3 = scene_mod.download([a * 3, b * 3])
    assert r3[0].base is blk2 or any(r3[0].base is e[1] for e in scene_mod._OUT_POOL)
    assert np.array_equal(r3[0], npa(a) * 3) and np.array_equal(r3[1], npa(b) * 3)
    r3[0][0, 0] = -1.0                       # caller-owned, writable


def test_work_item_claim_order_is_segment_major():
    """k_make_items: column 3 of the work items is a permutation of the
    items, every tile's first depth segment before any tile's second, tile
    order within a segment index (the persistent walk's claim order)."""
    import os

    os.environ["SDGR_SEG_LEN"] = "1024"   # many segments per tile (<= 64: beyond, identity order)
    try:
        tank = targets.composite_target(targets.tank_preset(), [30000, 12000, 4000], seed=2)
        cfg = sdgr.RadarConfig(azimuth_deg=20.0, elevation_deg=45.0, altitude_m=0.5, n_range=128, n_azimuth=128)
        fwd = sdgr.render_forward(tank, cfg)
        tl = fwd.rays
        ni = int(tl.n_items[0].item())
        it = tl.items[:ni].cpu().numpy()
    finally:
        del os.environ["SDGR_SEG_LEN"]
    assert ni > 0 and int(tl.n_items[1].item()) == 0
    order = it[:, 3]
    assert np.array_equal(np.sort(order), np.arange(ni))
    tile, start = it[:, 0], it[:, 1]
    first = {}
    for i in range(ni):                      # items are tile-major, segment-minor
        first.setdefault(int(tile[i]), i)
    seg = np.array([i - first[int(tile[i])] for i in range(ni)])
    k = seg[order]
    assert np.all(np.diff(k) >= 0)           # segment-major
    for kk in np.unique(k):                  # tile order within one segment index
        assert np.all(np.diff(tile[order[k == kk]]) > 0)
    assert np.any(seg > 0)


def test_host_copy_fallbacks():
    """Past the result-block cap, download() copies out of the staging block
    into fresh arrays; scene arrays that share a page with another registered
    array (registered or, where the driver refuses, staged) upload the same
    values, also after in-place updates."""
    import gc

    from paper_2506_21633_b200 import scene as scene_mod

    dev = torch.device("cuda", 0)
    a = torch.randn((400000, 3), dtype=torch.float64, device=dev)
    old, old_pool = scene_mod._OUT_POOL_BYTES, scene_mod._OUT_POOL[:]
    try:
        scene_mod._OUT_POOL_BYTES = 0            # no recycled blocks: the staging path
        scene_mod._OUT_POOL[:] = []
        r = scene_mod.download([a])
        assert np.array_equal(r[0], npa(a))
        assert r[0].flags.owndata and not scene_mod._OUT_POOL   # fresh memory, no block taken
    finally:
        scene_mod._OUT_POOL_BYTES = old
        scene_mod._OUT_POOL[:] = old_pool
    # two halves of one buffer share the page at their boundary
    big = np.random.default_rng(0).normal(size=(2 * 600000 + 3,))
    h1, h2 = big[: 600000 + 1], big[600000 + 1:]
    for _ in range(3):                           # second sighting registers, third reuses
        for h in (h1, h2):
            t = scene_mod.upload_f64(h, dev)
            assert np.array_equal(npa(t), h)
    states = [e[3] for e in scene_mod._SEEN.values() if e[0]() is big]
    assert len(states) == 2 and set(states) <= {"pinned", "failed"}, states   # the driver may accept the shared page
    h1[:] += 1.0                                 # in-place update seen through both paths
    h2[:] -= 1.0
    assert np.array_equal(npa(scene_mod.upload_f64(h1, dev)), h1)
    assert np.array_equal(npa(scene_mod.upload_f64(h2, dev)), h2)
    del h1, h2, big, t
    gc.collect()
