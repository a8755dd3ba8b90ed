"""The oracle (oracle/sdgr_oracle.py) pinned against the reference's own outputs.

tests/golden/*.npz were produced by running the reference sarsplat package
(tests/golden/make_golden.py).  With exp="numpy" the oracle's key chain is the
reference's operation for operation, so projection arrays and every pair list
must match BIT-FOR-BIT; compositing/gradients to ~1e-10.  With exp="device"
(the CUDA kernels' exp) keys must still match exactly.
"""
import numpy as np
import pytest

from conftest import GROUPS, assert_close, golden_files, load_golden
from oracle import sdgr_oracle as O

GOLDEN = golden_files()


def _cell_checksum(cell, prim_idx):
    h = np.uint64(1469598103934665603)
    x = (cell.astype(np.uint64) << np.uint64(32)) ^ prim_idx.astype(np.uint64)
    w = (np.arange(x.size, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) | np.uint64(1)
    with np.errstate(over="ignore"):
        return np.uint64(h ^ np.bitwise_xor.reduce(x * w)) if x.size else h


@pytest.mark.parametrize("path", GOLDEN, ids=[p.stem for p in GOLDEN])
def test_oracle_matches_reference_golden(path):
    z, scene, cfg, cutoff = load_golden(path)
    f = O.render_forward(scene, cfg, cutoff=cutoff, exp="numpy")
    p = f.proj
    assert np.array_equal(p.indices, z["indices"])
    assert p.n_culled == int(z["n_culled"]) and p.n_skipped == int(z["n_skipped"])
    for k in ("uv_comp", "uv_img", "depth"):
        assert np.array_equal(getattr(p, k), z[k]), k
    assert np.array_equal(p.cov_comp[:, [0, 0, 1], [0, 1, 1]], z["cov_comp"])
    assert np.array_equal(p.cov_img[:, [0, 0, 1], [0, 1, 1]], z["cov_img"])
    for plane, pairs in ((0, f.rays), (1, f.spl)):
        assert len(pairs.cell) == int(z[f"pairs{plane}_count"])
        assert _cell_checksum(pairs.cell, p.indices[pairs.prim]) == z[f"pairs{plane}_checksum"]
        if f"pairs{plane}_cell" in z:
            assert np.array_equal(pairs.cell, z[f"pairs{plane}_cell"])
            assert np.array_equal(p.indices[pairs.prim], z[f"pairs{plane}_prim"])
        tt, gi, rg = O.tile_lists(pairs, p, plane)
        assert np.array_equal(tt, z[f"tiles{plane}_tile"])
        assert np.array_equal(gi, z[f"tiles{plane}_prim"])
        assert np.array_equal(rg, z[f"tiles{plane}_range"])
    assert_close(f.inten.intensity, z["intensity"], atol=1e-12, rtol=1e-10, what="intensity")
    assert_close(f.image, z["image"], atol=1e-12, rtol=1e-10, what="image")
    rows = z["grad_rows"]
    for tag, dlds in (("n", z["dLdS"]), ("s", z["image"])):
        g = O.backward(f, dlds)
        for k in GROUPS + ("uv_grad_norm",):
            assert_close(g[k][rows], z[f"g{tag}_{k}"], atol=1e-11, rtol=1e-9, what=f"{k} ({tag})")
        assert np.array_equal(g["visible"][rows], z[f"g{tag}_visible"])


@pytest.mark.parametrize("path", [p for p in GOLDEN if "small" in p.stem or "perturbed" in p.stem],
                         ids=lambda p: p.stem)
def test_device_exp_keys_unchanged(path):
    """The device exp differs from numpy's by <= 1 ulp; no key may move."""
    z, scene, cfg, cutoff = load_golden(path)
    f = O.render_forward(scene, cfg, cutoff=cutoff, exp="device")
    for plane, pairs in ((0, f.rays), (1, f.spl)):
        tt, gi, rg = O.tile_lists(pairs, f.proj, plane)
        assert np.array_equal(gi, z[f"tiles{plane}_prim"])
        assert _cell_checksum(pairs.cell, f.proj.indices[pairs.prim]) == z[f"pairs{plane}_checksum"]


def test_oracle_exp_accuracy():
    x = np.linspace(np.log(0.001), np.log(5.0), 20001)
    got = np.array([O.oracle_exp(v) for v in x])
    ref = np.exp(x.astype(np.longdouble)).astype(np.float64)
    ulp = np.abs(got - ref) / np.spacing(ref)
    assert ulp.max() <= 1.0


def test_forward_known_answers():
    """Hand values of the reference's own stage tests (test_forward.py:138-158,
    test_backward.py:80-101): one / two stacked point-like scatterers."""
    from paper_2506_21633_b200.radar import RadarConfig
    from paper_2506_21633_b200.scene import Scene

    cfg = RadarConfig(azimuth_deg=20.0, elevation_deg=40.0, altitude_m=2.0, range_res_m=0.5,
                      azimuth_res_m=0.5, n_range=16, n_azimuth=16)
    view = O.make_view(cfg)
    # build a projection by hand: identity-like tiny covariance, kappa = 1, P = 1
    k = 2
    eye = np.broadcast_to(np.eye(2) * 1e-6, (k, 2, 2)).copy()
    proj = O.OracleProjection(
        indices=np.arange(k), uv_comp=np.array([[4.0, 4.0], [4.0, 4.0]]), depth=np.array([1.0, 2.0]),
        uv_img=np.array([[4.0, 4.0], [4.0, 4.0]]), cov_comp=eye, cov_img=eye.copy(), phase=np.ones(k),
        phase_unclamped=np.ones(k), ke_fwd=np.full(k, 0.5), ke_bwd=np.full(k, 0.5),
        look_dirs=np.tile([0.0, 0.0, 1.0], (k, 1)), look_dists=np.ones(k), view=view, n_scene=k,
        n_culled=0, n_skipped=0, cutoff=3.0)
    rays = O.ray_pairs(proj)
    it = O.intensities(rays, proj)
    assert it.intensity[0] == pytest.approx(1.0 - np.exp(-1.0), abs=1e-9)
    assert it.intensity[1] == pytest.approx((1.0 - np.exp(-1.0)) * np.exp(-1.0), abs=1e-9)
    del Scene


def test_naive_oracle_matches_golden_dense():
    """The naive loop renderer (render_reference restatement) reproduces the
    reference's dense-mode goldens (cutoff = inf), like criterion 2."""
    from oracle import sdgr_oracle as O
    for path in [p for p in GOLDEN if p.stem.endswith("_dense")]:
        z, scene, cfg, cutoff = load_golden(path)
        img = O.render_reference(scene, cfg)
        assert np.abs(img - z["image"]).max() <= 1e-10 * max(1.0, float(z["image"].max())), path.stem
