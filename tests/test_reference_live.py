"""Oracle vs the live reference package (build container only).

Imports sarsplat from /root/reference/pkg/src -- absent on the GPU box, where
these tests skip and the committed goldens carry the pin instead.  Random
scenes (the reference's own gradcheck generator) at several views: the
oracle's projection and pair lists must be bit-identical to the reference's,
images and gradients equal to ~1e-10.
"""
import sys

import numpy as np
import pytest

from conftest import GROUPS, REFERENCE_SRC, assert_close, has_reference

pytestmark = pytest.mark.reference
if not has_reference():
    pytest.skip("reference sources not present (GPU box)", allow_module_level=True)

sys.path.insert(0, str(REFERENCE_SRC))
import sarsplat as ss  # noqa: E402
from sarsplat.gradcheck import gradcheck_config, random_scene  # noqa: E402

from oracle import sdgr_oracle as O  # noqa: E402


@pytest.mark.parametrize("seed", range(8))
def test_oracle_equals_reference(seed):
    rng = np.random.default_rng(1000 + seed)
    scene = random_scene(rng, 6 + 5 * seed)
    cfg = gradcheck_config(rng, size=16 + 8 * (seed % 3))
    cutoff = np.inf if seed % 2 else 3.0
    fr = ss.render_forward(scene, cfg, cutoff=cutoff)
    fo = O.render_forward(scene, cfg, cutoff=cutoff, exp="numpy")
    p, q = fr.projection, fo.proj
    for k in ("indices", "uv_comp", "uv_img", "depth", "cov_comp", "cov_img"):
        assert np.array_equal(getattr(p, k), getattr(q, k)), k
    assert np.array_equal(fr.rays.pair_cell, fo.rays.cell)
    assert np.array_equal(fr.rays.pair_prim, fo.rays.prim)
    assert np.array_equal(fr.splat.pair_pixel, fo.spl.cell)
    assert np.array_equal(fr.splat.pair_prim, fo.spl.prim)
    assert_close(fo.image, fr.image, atol=1e-13, rtol=1e-11, what="image")
    g = rng.normal(size=fr.image.shape)
    gr = ss.backward(fr, g)
    go = O.backward(fo, g)
    for k in GROUPS + ("uv_grad_norm",):
        assert_close(go[k], getattr(gr, k), atol=1e-12, rtol=1e-9, what=k)
    assert np.array_equal(go["visible"], gr.visible)


def test_targets_port_matches_reference():
    from paper_2506_21633_b200 import targets as T

    a = ss.composite_target(ss.tank_preset(), [3000, 1500, 500], seed=11)
    b = T.composite_target(T.tank_preset(), [3000, 1500, 500], seed=11)
    for k in GROUPS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    a = ss.building_scene(ss.CuboidSpec(height=5, width=4, length=6), ground_extent=12, density=2.0, seed=3)
    b = T.building_scene(T.CuboidSpec(5, 4, 6), 12, 2.0, seed=3)
    for k in GROUPS:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_view_constants_equal_reference():
    from paper_2506_21633_b200.radar import RadarConfig, view_constants
    from sarsplat.geometry import (computation_jacobian, imaging_jacobian, radar_position,
                                   radar_rotation, radar_translation)

    for az, el, alt in ((0.0, 45.0, 1000.0), (37.0, 15.0, 0.5), (301.5, 72.0, 3.0)):
        rc = ss.RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=alt, n_range=96, n_azimuth=160,
                            ray_grid=(120, 80))
        mc = RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=alt, n_range=96, n_azimuth=160,
                         ray_grid=(120, 80))
        v = view_constants(mc)
        R = radar_rotation(az, el)
        assert np.array_equal(np.array(v.R).reshape(3, 3), R)
        assert np.array_equal(np.array(v.T), radar_translation(rc))
        assert np.array_equal(np.array(v.cam), radar_position(rc))
        assert np.array_equal(np.array(v.mc).reshape(2, 3), computation_jacobian(rc) @ R)
        assert np.array_equal(np.array(v.mi).reshape(2, 3), imaging_jacobian(rc) @ R)
