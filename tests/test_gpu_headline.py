"""Parity at the benchmarked configurations (B200 only).

BASELINE.json's metric is quoted on SURVEY.md §8d c4: 16 tanks on a 4x4
grid (20 m pitch), 1 000 000 Gaussians, 512x512 views at el 30/45/60.  This
module checks, on that exact scene, both device paths against the oracle
(oracle/sdgr_oracle.py, pinned to the reference's own outputs):

  * the single-view drop-in: render_forward(host FP64 scene) + backward
    (reference forward.py:256-273, backward.py:243-290), one view per
    elevation;
  * the benchmarked path: MultiViewStep with FP32 device parameters, one
    batched launch per stage, 8 view lanes, s_stop = 40 and depth segments of
    >= 2048 Gaussians -- its accumulated gradients against the sum of the
    oracle's per-view gradients;

and the single-view drop-in on c3 (single 300k tank, 256x256) at el 15 and
75, where tile lists reach ~160k Gaussians.

The oracle runs with the reference's own numpy exp (exp="numpy"), so the
bit-exact tile key lists also tie the device key chain to the reference's
arithmetic at 1M Gaussians.  Bar: key lists and tile ranges bit-exact, image,
intensities and every gradient column within 1e-6 + 1e-4 |ref|, visible exact.
"""
import numpy as np
import pytest

from conftest import GROUPS, assert_close, npa

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200 import targets  # noqa: E402
from oracle import sdgr_oracle as O  # noqa: E402

C4_VIEWS = ((36.0, 30.0), (150.0, 45.0), (267.0, 60.0))   # on bench.py's az 0:360:3 x el grid
C3_VIEWS = ((0.0, 15.0), (45.0, 75.0))


def c4_config(az, el, size=512):
    return sdgr.RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=0.5, range_res_m=0.3,
                            azimuth_res_m=0.3, n_range=size, n_azimuth=size)


@pytest.fixture(scope="module")
def c4_scene():
    # float32-exact: the FP32 device scene of the bench and the FP64 host scene
    # of the drop-in describe the same Gaussians
    return targets.to_float32_exact(targets.tank_grid(1_000_000))


_ORACLE = {}


def oracle_view(scene, key, cfg, seed):
    """Oracle forward + backward of one view (cached per module run)."""
    if key not in _ORACLE:
        fo = O.render_forward(scene, cfg, exp="numpy")
        dlds = np.random.default_rng(seed).normal(size=fo.image.shape)
        _ORACLE[key] = (fo, dlds, O.backward(fo, dlds))
    return _ORACLE[key]


def check_tiles(tl, fo, plane, what):
    tt, gi, rg = O.tile_lists(fo.rays if plane == 0 else fo.spl, fo.proj, plane)
    n = tl.n_pairs
    assert n == tt.size, (what, n, tt.size)
    assert np.array_equal(tl.pair_tile[:n].cpu().numpy().astype(np.int64), tt), what
    assert np.array_equal(tl.tile_prim[:n].cpu().numpy().astype(np.int64), gi), what
    assert np.array_equal(tl.tile_range.cpu().numpy().astype(np.int64), rg), what


def dropin_vs_oracle(scene, cfg, key, seed):
    fo, dlds, go = oracle_view(scene, key, cfg, seed)
    fwd = sdgr.render_forward(scene, cfg)
    p = fwd.projection
    assert np.array_equal(npa(p.indices), fo.proj.indices)
    assert p.n_culled == fo.proj.n_culled and p.n_skipped == fo.proj.n_skipped
    # the FP64 key chain on every visible Gaussian: pixel centres and depth
    # bit-identical to the reference's arithmetic (none of them involves exp)
    assert np.array_equal(npa(p.uv_comp), fo.proj.uv_comp), key
    assert np.array_equal(npa(p.uv_img), fo.proj.uv_img), key
    assert np.array_equal(npa(p.depth), fo.proj.depth), key
    check_tiles(fwd.rays, fo, 0, f"{key} comp tiles")
    check_tiles(fwd.splat, fo, 1, f"{key} img tiles")
    assert_close(npa(fwd.intensities.intensity), fo.inten.intensity, what=f"{key} intensity")
    assert_close(fwd.image, fo.image, what=f"{key} image")
    g = sdgr.backward(fwd, dlds)
    for k in GROUPS + ("uv_grad_norm",):
        assert_close(getattr(g, k), go[k], what=f"{key} grad {k}")
    assert np.array_equal(g.visible, go["visible"])
    return fwd


@pytest.mark.parametrize("az,el", C4_VIEWS, ids=[f"el{int(e)}" for _, e in C4_VIEWS])
def test_c4_dropin_vs_oracle(c4_scene, az, el):
    """Headline scene, one view: render_forward(host scene) + backward(N(0,1))."""
    fwd = dropin_vs_oracle(c4_scene, c4_config(az, el), ("c4", az, el), seed=int(el))
    if el == 45.0:
        # dL/dS = S (gradcheck.py:79): the gradcheck-style upstream gradient
        fo, _, _ = _ORACLE[("c4", az, el)]
        go = O.backward(fo, fo.image)
        g = sdgr.backward(fwd, fwd.image)
        for k in GROUPS + ("uv_grad_norm",):
            assert_close(getattr(g, k), go[k], what=f"dL/dS=S grad {k}")


@pytest.mark.parametrize("order", ["native", "morton"])
def test_c4_benchmarked_step_vs_oracle(c4_scene, order):
    """The exact path bench.py times (MultiViewStep: FP32 parameters, batched
    K1-K5, 8 lanes, s_stop 40, >= 2048-Gaussian depth segments) on the three
    c4 views: accumulated gradients == sum of the oracle's per-view gradients.
    "morton": the scene in spatial_order, as bench.py stores it; its gradients
    are the oracle's (computed on the sampler's order) permuted."""
    from paper_2506_21633_b200.multiview import MULTIVIEW_SEG_LEN, MultiViewStep

    cfgs = [c4_config(az, el) for az, el in C4_VIEWS]
    ref = {k: 0.0 for k in GROUPS + ("uv_grad_norm",)}
    vis = 0
    dls = []
    for (az, el), c in zip(C4_VIEWS, cfgs):
        _, dlds, go = oracle_view(c4_scene, ("c4", az, el), c, seed=int(el))
        dls.append(dlds)
        for k in ref:
            ref[k] = ref[k] + go[k]
        vis = vis + go["visible"].astype(np.int64)
    scene = c4_scene
    if order == "morton":
        scene, perm = sdgr.spatial_sort(c4_scene)
        assert not np.array_equal(perm, np.arange(len(perm)))
        ref = {k: v[perm] for k, v in ref.items()}
        vis = vis[perm]
    ds = sdgr.DeviceScene.from_host(scene, dtype=torch.float32)
    step = MultiViewStep(ds, cfgs)
    assert step.s_stop == sdgr.S_STOP and step.n_lanes == len(cfgs)
    got = step.run(torch.from_numpy(np.stack(dls)).cuda())
    assert all(t.seg_len >= MULTIVIEW_SEG_LEN for t in step.slot_tiles)
    for k in ref:
        assert_close(getattr(got, k).double().cpu().numpy(), ref[k], what=f"step grad {k}")
    assert np.array_equal(got.visible.cpu().numpy().astype(np.int64), vis)


@pytest.fixture(scope="module")
def c3_scene():
    return targets.composite_target(targets.tank_preset(), [180000, 90000, 30000], seed=3)


@pytest.mark.parametrize("az,el", C3_VIEWS, ids=[f"el{int(e)}" for _, e in C3_VIEWS])
def test_c3_dropin_vs_oracle(c3_scene, az, el):
    """Single 300k tank at 256x256: the deepest tile lists."""
    dropin_vs_oracle(c3_scene, c4_config(az, el, size=256), ("c3", az, el), seed=100 + int(el))


def test_c5_large_footprints_vs_oracle():
    """SURVEY §8d c5 at sigma = 1.0 m (~320 member cells per Gaussian): every
    footprint is wider than the 8x8 cell window, so K1's tile test, the
    walks' member masks and the splat run their exact FP64 per-cell loops."""
    scene = targets.tank_grid(10_000)
    scene.log_scales[:] = np.log(1.0)
    scene = targets.to_float32_exact(scene)
    dropin_vs_oracle(scene, c4_config(150.0, 45.0), ("c5", 1.0), seed=5)
