"""Host-side logic that needs no GPU: view constants, config validation,
depth-key encoding, work-item sizing, error classes, scene generators."""
import math

import numpy as np
import pytest

from conftest import GROUPS, golden_files, load_golden


def test_view_constants_match_oracle_bitwise():
    from oracle import sdgr_oracle as O
    from paper_2506_21633_b200.radar import RadarConfig, view_constants

    for az, el, alt, nr, na, rg in ((0.0, 45.0, 1000.0, 128, 128, None), (37.0, 15.0, 0.5, 256, 256, None),
                                    (301.5, 72.0, 3.0, 96, 160, (120, 80))):
        cfg = RadarConfig(azimuth_deg=az, elevation_deg=el, altitude_m=alt, n_range=nr, n_azimuth=na, ray_grid=rg)
        v = view_constants(cfg)
        o = O.make_view(cfg)
        assert np.array_equal(np.array(v.R).reshape(3, 3), o.R)
        assert np.array_equal(np.array(v.T), o.T)
        assert np.array_equal(np.array(v.cam), o.cam)
        assert np.array_equal(np.array(v.mc).reshape(2, 3), o.mc)
        assert np.array_equal(np.array(v.mi).reshape(2, 3), o.mi)
        assert (v.den_u, v.den_v, v.off_vi) == (o.den_u, o.den_v, o.off_vi)
        assert (v.n_u, v.n_v, v.n_az, v.n_rg) == (o.n_u, o.n_v, o.n_az, o.n_rg)


def test_radar_config_validation():
    from paper_2506_21633_b200 import InvalidParameterError, RadarConfig

    with pytest.raises(InvalidParameterError):
        RadarConfig(azimuth_deg=0.0, elevation_deg=90.0)
    with pytest.raises(InvalidParameterError):
        RadarConfig(azimuth_deg=0.0, elevation_deg=45.0, range_res_m=0.0)
    with pytest.raises(InvalidParameterError):
        RadarConfig(azimuth_deg=float("nan"), elevation_deg=45.0)
    c = RadarConfig(azimuth_deg=10.0, elevation_deg=30.0, n_range=64, n_azimuth=32)
    assert c.n_rays == (32, 64)
    assert c.with_view(20.0, 40.0).azimuth_deg == 20.0


def test_view_constants_reject_oversized_planes():
    from paper_2506_21633_b200 import InvalidParameterError, RadarConfig
    from paper_2506_21633_b200.radar import view_constants

    with pytest.raises(InvalidParameterError):
        view_constants(RadarConfig(azimuth_deg=0.0, elevation_deg=45.0, n_range=40000, n_azimuth=8))
    with pytest.raises(InvalidParameterError):
        view_constants(RadarConfig(azimuth_deg=0.0, elevation_deg=45.0), cutoff=float("nan"))


def test_depth_key_encoding_is_order_preserving():
    """The device key (common.cuh:depth_key) restated in numpy: sorting keys
    stably must reproduce np.lexsort((index, depth)) incl. -0.0 == 0.0 ties."""
    import torch

    from paper_2506_21633_b200.rasterizer import decode_depth

    rng = np.random.default_rng(0)
    d = np.concatenate([rng.normal(size=4000), [0.0, -0.0, 0.0, 1e-300, -1e-300, 5.0, 5.0, -7.0]])
    dd = np.where(d == 0.0, 0.0, d)
    b = dd.view(np.uint64)
    key = np.where(b >> np.uint64(63) == 1, ~b, b | np.uint64(1 << 63))
    order = np.argsort(key, kind="stable")
    assert np.array_equal(order, np.lexsort((np.arange(d.size), d)))
    back = decode_depth(torch.from_numpy(key.view(np.int64))).numpy()
    assert np.array_equal(back, dd)


def test_segment_length_heuristic():
    from paper_2506_21633_b200.rasterizer import _seg_len

    assert _seg_len(0) == 256 and _seg_len(1000) == 256
    assert _seg_len(1_310_000) % 256 == 0 and 256 <= _seg_len(1_310_000) <= 1024
    assert _seg_len(10**9) == 8192


def test_shard_views_partition():
    from paper_2506_21633_b200.multiview import shard_views

    views = list(range(360))
    for world in (1, 2, 4, 8):
        shards = [shard_views(views, r, world) for r in range(world)]
        assert sorted(sum(shards, [])) == views
        assert all(len(s) == 360 // world for s in shards)


def test_error_hierarchy_mirrors_reference():
    from paper_2506_21633_b200 import errors as E

    assert issubclass(E.InvalidParameterError, ValueError)
    assert issubclass(E.NumericalError, ArithmeticError)
    assert issubclass(E.DegenerateProjectionError, ArithmeticError)
    assert issubclass(E.StateError, RuntimeError)
    for cls in (E.InvalidParameterError, E.NumericalError, E.StateError, E.DivergenceError):
        assert issubclass(cls, E.SarsplatError)


@pytest.mark.parametrize("path", [p for p in golden_files() if "tank" in p.stem][:1], ids=lambda p: p.stem)
def test_targets_port_reproduces_golden_scene(path):
    from paper_2506_21633_b200 import targets

    z, scene, _, _ = load_golden(path)
    s = targets.composite_target(targets.tank_preset(), [6000, 3000, 1000], seed=3)
    for k in GROUPS:
        assert np.array_equal(getattr(s, k), z[f"scene_{k}"]), k


def test_tank_grid_layout():
    from paper_2506_21633_b200 import targets

    s = targets.tank_grid(n_total=16_000, grid=4, pitch=20.0)
    assert len(s) == 16_000
    cx = np.sort(np.unique(np.round(s.positions[:, 0] / 20.0)))
    assert cx.min() >= -2 and cx.max() <= 2
    f = targets.to_float32_exact(s)
    assert np.array_equal(f.positions, f.positions.astype(np.float32).astype(np.float64))


def test_package_imports_without_gpu():
    import paper_2506_21633_b200 as sdgr

    assert sdgr.__version__
    assert callable(sdgr.render) and callable(sdgr.backward)
    assert math.isfinite(sdgr.S_STOP)


def test_scene_descriptor_validation():
    """a DeviceScene with mixed dtypes, wrong shapes or
    non-contiguous arrays is rejected before any pointer reaches a kernel
    (CPU tensors are rejected too)."""
    import pytest
    import torch

    from paper_2506_21633_b200.errors import InvalidParameterError
    from paper_2506_21633_b200.rasterizer import _scene_desc
    from paper_2506_21633_b200.scene import DeviceScene

    def mk(dtypes=(torch.float32,) * 5, n=4):
        return DeviceScene(*(torch.zeros((n, w), dtype=dt) for w, dt in zip((3, 4, 3, 16, 2), dtypes)))

    with pytest.raises(InvalidParameterError, match="CUDA"):
        _scene_desc(mk())
    with pytest.raises(InvalidParameterError, match="dtype"):
        _scene_desc(mk((torch.float32, torch.float64, torch.float32, torch.float32, torch.float32)))
    bad = mk()
    bad.sh_coeffs = torch.zeros((16, 4)).T            # transposed view: right shape, not contiguous
    with pytest.raises(InvalidParameterError, match="contiguous"):
        _scene_desc(bad)
    bad = mk()
    bad.ke_raw = torch.zeros((4, 3))
    with pytest.raises(InvalidParameterError, match="shape"):
        _scene_desc(bad)


def test_spatial_order_is_a_morton_permutation():
    import paper_2506_21633_b200 as sdgr

    rng = np.random.default_rng(0)
    pos = rng.uniform(-5, 5, size=(5000, 3))
    perm = sdgr.spatial_order(pos)
    assert np.array_equal(np.sort(perm), np.arange(len(pos)))
    # neighbours in the new order are close in space (Z-curve locality)
    d_sorted = np.linalg.norm(np.diff(pos[perm], axis=0), axis=1).mean()
    d_orig = np.linalg.norm(np.diff(pos, axis=0), axis=1).mean()
    assert d_sorted < 0.2 * d_orig
    scene = sdgr.Scene(pos, rng.normal(size=(5000, 4)), rng.normal(size=(5000, 3)),
                       rng.normal(size=(5000, 16)), rng.normal(size=(5000, 2)))
    s2, p2 = sdgr.spatial_sort(scene)
    assert np.array_equal(p2, perm)
    for k in ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw"):
        assert np.array_equal(getattr(s2, k), getattr(scene, k)[perm])
    # degenerate inputs: empty, one point, non-finite rows keep a valid permutation
    assert sdgr.spatial_order(np.zeros((0, 3))).shape == (0,)
    assert np.array_equal(sdgr.spatial_order(np.zeros((1, 3))), [0])
    bad = pos[:10].copy()
    bad[3] = np.nan
    assert np.array_equal(np.sort(sdgr.spatial_order(bad)), np.arange(10))
