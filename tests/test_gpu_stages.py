"""The reference's stage API on the device (B200 only).

* a7 `_footprint_pairs` / the CSR of `build_ray_lists` and `_build_splat_pairs`
  (forward.py:60-155, 213-224): the device per-cell member pairs
  (sdgr_cell_pairs) against every reference golden -- full (cell, scene
  index) lists where the golden stores them, count + order-sensitive
  checksum elsewhere (tests/golden/make_golden.py:34-41, 91-95).
* The reference-shaped views (RayLists, SplatPairs, IntensityBuffer) and the
  stage tuples of backward.py:86-240 against the oracle.
* The reference's own known-answer tests (tests/test_forward.py:82-233,
  tests/test_backward.py:31-101), ported to the device path through a
  synthetic Projection (Projection.from_planes, the device counterpart of
  test_forward.synthetic_projection).
"""
import math

import numpy as np
import pytest

from conftest import GROUPS, assert_close, golden_files, load_golden, npa

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200 import targets  # noqa: E402
from oracle import sdgr_oracle as O  # noqa: E402

GOLDEN = golden_files()


def checksum(cell, prim_idx):
    """tests/golden/make_golden.py:34-41 (order-sensitive 64-bit fold)."""
    h = np.uint64(1469598103934665603)
    x = (cell.astype(np.uint64) << np.uint64(32)) ^ prim_idx.astype(np.uint64)
    w = (np.arange(x.size, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) | np.uint64(1)
    with np.errstate(over="ignore"):
        return np.uint64(h ^ np.bitwise_xor.reduce(x * w)) if x.size else h


@pytest.mark.parametrize("path", GOLDEN, ids=[p.stem for p in GOLDEN])
def test_cell_pairs_match_reference_goldens(path):
    z, scene, cfg, cutoff = load_golden(path)
    fwd = sdgr.render_forward(scene, cfg, cutoff=cutoff)
    for plane, tl in ((0, fwd.rays), (1, fwd.splat)):
        c = tl.cells()
        cell = c["cell"].cpu().numpy()
        prim = c["prim"].cpu().numpy()
        assert cell.size == int(z[f"pairs{plane}_count"]), (plane, cell.size)
        if f"pairs{plane}_cell" in z:
            assert np.array_equal(cell, z[f"pairs{plane}_cell"])
            assert np.array_equal(prim, z[f"pairs{plane}_prim"])
        assert checksum(cell, prim) == z[f"pairs{plane}_checksum"], plane


def _random_case(seed=3, n=40, cutoff=3.0):
    rng = np.random.default_rng(seed)
    scene = targets.random_scene(rng, n, spread=3.0)
    cfg = sdgr.RadarConfig(azimuth_deg=50.0, elevation_deg=45.0, altitude_m=2.0, range_res_m=0.25,
                           azimuth_res_m=0.25, n_range=40, n_azimuth=48)
    return scene, cfg, rng


@pytest.mark.parametrize("cutoff", [3.0, math.inf], ids=["cut", "dense"])
def test_reference_views_vs_oracle(cutoff):
    """RayLists / SplatPairs / IntensityBuffer fields (forward.py:112-210)."""
    scene, cfg, _ = _random_case(cutoff=cutoff)
    fwd = sdgr.render_forward(scene, cfg, cutoff=cutoff)
    fo = O.render_forward(scene, cfg, cutoff=cutoff, exp="device")
    r, o = fwd.rays, fo.rays
    assert isinstance(r.pair_cell, np.ndarray)          # host callers get numpy, like the reference
    assert len(r) == o.cell.size
    assert np.array_equal(r.pair_cell, o.cell) and np.array_equal(r.pair_prim, o.prim)
    assert np.array_equal(r.offsets, o.offsets)
    assert np.array_equal(r.delta[:, 0], o.dx) and np.array_equal(r.delta[:, 1], o.dy)
    assert np.array_equal(r.q, o.q)
    assert_close(r.weight, o.w, atol=1e-15, rtol=1e-14, what="weight")
    iu, iv = 24, 20
    assert np.array_equal(r.cell_list(iu, iv), o.prim[o.offsets[iv * cfg.n_azimuth + iu]:
                                                       o.offsets[iv * cfg.n_azimuth + iu + 1]])
    s, so = fwd.splat, fo.spl
    assert np.array_equal(s.pair_pixel, so.cell) and np.array_equal(s.pair_prim, so.prim)
    b, bo = fwd.intensities, fo.inten
    for k in ("tau", "trans", "absorb", "contrib"):
        assert_close(getattr(b, k), getattr(bo, k), atol=1e-14, rtol=1e-12, what=k)
    assert_close(b.intensity, bo.intensity, what="intensity")


def test_stage_tuples_vs_oracle():
    """grad_image_stage / grad_intensity_stage / grad_geometry_stage /
    grad_sh_stage return the reference's tuples (backward.py:86-240)."""
    scene, cfg, rng = _random_case(seed=5, n=30)
    fwd = sdgr.render_forward(scene, cfg)
    fo = O.render_forward(scene, cfg, exp="device")
    dl = rng.normal(size=fwd.image.shape)
    go = O.backward(fo, dl, stages=True)
    st = go["_stages"]
    dI, dbeta, dcov_i, duv_i = sdgr.grad_image_stage(fwd, dl)
    assert_close(dI, st["dI"], what="dL/dI")
    assert_close(dcov_i, st["dcov_i"], what="dL/dcov_img")
    assert_close(duv_i, st["duv_i"], what="dL/duv_img")
    want_beta = dl.reshape(-1)[fo.spl.cell] * fo.inten.intensity[fo.spl.prim]
    assert_close(dbeta, want_beta, what="dL/dbeta")
    dP, dke, dcov_c, duv_c = sdgr.grad_intensity_stage(fwd, dI)
    assert_close(dP, st["dP"], what="dL/dP")
    assert_close(dke, st["dke"], what="dL/dke_sum")
    assert_close(dcov_c, st["dcov_c"], what="dL/dcov_comp")
    assert_close(duv_c, st["duv_c"], what="dL/duv_comp")
    idx = fo.proj.indices
    dpos, drot, dlogs = sdgr.grad_geometry_stage(fwd, dcov_c, dcov_i, duv_c, duv_i, dP)
    assert_close(dpos, go["positions"][idx], what="dL/dpos")
    assert_close(drot, go["rotations"][idx], what="dL/drot")
    assert_close(dlogs, go["log_scales"][idx], what="dL/dlogs")
    assert_close(sdgr.grad_sh_stage(fwd, dP), go["sh_coeffs"][idx], what="dL/dsh")


# ------------------------------------------------ ported reference KATs ------
def tiny_config(n=16, el=40.0):
    """tests/test_forward.py:35-40."""
    return sdgr.RadarConfig(azimuth_deg=20.0, elevation_deg=el, altitude_m=2.0, range_res_m=0.5,
                            azimuth_res_m=0.5, n_range=n, n_azimuth=n)


def synthetic_projection(uv_comp, depth, cov=None, ke_sum=None, phase=None, config=None):
    """tests/test_forward.py:43-59 on the device: identity covariances,
    kappa = P = 1 by default, uv_img = uv_comp, cutoff 3."""
    return sdgr.Projection.from_planes(config or tiny_config(), np.asarray(uv_comp, float), np.asarray(depth, float),
                                       cov_comp=cov, ke_sum=ke_sum, phase=phase, cutoff=3.0)


def test_kat_depth_sort_order_and_ties():
    rays = sdgr.build_ray_lists(synthetic_projection([[4.0, 4.0], [4.0, 4.0]], depth=[2.0, 1.0]))
    assert list(rays.cell_list(4, 4)) == [1, 0]            # shallower first (test_forward.py:82-86)
    rays = sdgr.build_ray_lists(synthetic_projection([[4.0, 4.0]] * 3, depth=[1.0, 1.0, 1.0]))
    assert list(rays.cell_list(4, 4)) == [0, 1, 2]         # ties by index (:88-91)


def test_kat_membership_matches_brute_force(rng):
    """test_forward.py:93-111."""
    k = 12
    uv = rng.uniform(-2.0, 17.0, size=(k, 2))
    cov = np.empty((k, 2, 2))
    for i in range(k):
        a = rng.normal(size=(2, 2))
        cov[i] = a @ a.T + 0.3 * np.eye(2)
    proj = synthetic_projection(uv, depth=rng.uniform(0, 5, k), cov=cov)
    rays = sdgr.build_ray_lists(proj)
    inv = np.linalg.inv(cov)
    for iv in range(16):
        for iu in range(16):
            d = np.array([iu, iv]) - uv
            expected = [i for i in range(k) if d[i] @ inv[i] @ d[i] <= 9.0]
            assert sorted(rays.cell_list(iu, iv).tolist()) == expected, (iu, iv)


def test_kat_point_footprint_rule():
    """test_forward.py:113-123: a tiny footprint between cell centres covers
    nothing; centred on a cell it covers exactly that cell."""
    cov = np.eye(2)[None] * 1e-6
    assert len(sdgr.build_ray_lists(synthetic_projection([[4.5, 4.5]], depth=[1.0], cov=cov))) == 0
    rays = sdgr.build_ray_lists(synthetic_projection([[4.0, 4.0]], depth=[1.0], cov=cov))
    assert len(rays) == 1 and rays.cell_list(4, 4).tolist() == [0]


def test_kat_depth_nondecreasing_in_every_cell(rng):
    k = 30
    proj = synthetic_projection(rng.uniform(0, 15, size=(k, 2)), depth=rng.uniform(0, 5, k))
    rays = sdgr.build_ray_lists(proj)
    depth, off, prim = proj.depth, rays.offsets, rays.pair_prim
    for c in range(rays.n_u * rays.n_v):
        assert np.all(np.diff(depth[prim[off[c]:off[c + 1]]]) >= 0)


def test_kat_single_ray_and_stacked_intensities():
    """test_forward.py:138-158: I = 1 - e^-1 and (1 - e^-1) e^-1."""
    cov = np.eye(2)[None] * 1e-6
    proj = synthetic_projection([[4.0, 4.0]], depth=[1.0], cov=cov)
    buf = sdgr.compute_intensities(sdgr.build_ray_lists(proj), proj)
    assert buf.intensity[0] == pytest.approx(1.0 - np.exp(-1.0), abs=1e-9)
    proj = synthetic_projection([[4.0, 4.0]], depth=[1.0], cov=cov, ke_sum=[0.0])
    assert sdgr.compute_intensities(sdgr.build_ray_lists(proj), proj).intensity[0] == 0.0
    cov2 = np.broadcast_to(np.eye(2) * 1e-6, (2, 2, 2)).copy()
    proj = synthetic_projection([[4.0, 4.0], [4.0, 4.0]], depth=[1.0, 2.0], cov=cov2)
    buf = sdgr.compute_intensities(sdgr.build_ray_lists(proj), proj)
    assert buf.intensity[0] == pytest.approx(1.0 - np.exp(-1.0), abs=1e-9)
    assert buf.intensity[1] == pytest.approx((1.0 - np.exp(-1.0)) * np.exp(-1.0), abs=1e-9)


def test_kat_transmittance_monotone_and_energy_bound(rng):
    """test_forward.py:160-182."""
    k = 25
    proj = synthetic_projection(rng.uniform(0, 15, size=(k, 2)), depth=rng.uniform(0, 5, k),
                                ke_sum=rng.uniform(0.1, 3.0, k))
    rays = sdgr.build_ray_lists(proj)
    buf = sdgr.compute_intensities(rays, proj)
    off = rays.offsets
    for c in range(rays.n_u * rays.n_v):
        assert np.all(np.diff(buf.trans[off[c]:off[c + 1]]) <= 1e-15)
    phase = rng.uniform(0.2, 2.5, 20)
    proj = synthetic_projection(rng.uniform(0, 15, size=(20, 2)), depth=rng.uniform(0, 5, 20),
                                ke_sum=rng.uniform(0.1, 4.0, 20), phase=phase)
    rays = sdgr.build_ray_lists(proj)
    buf = sdgr.compute_intensities(rays, proj)
    per_ray = np.bincount(rays.pair_cell, weights=buf.contrib, minlength=rays.n_u * rays.n_v)
    assert per_ray.max() <= phase.max() + 1e-12


def test_kat_nonfinite_names_primitive():
    """test_forward.py:184-189."""
    proj = synthetic_projection([[4.0, 4.0]], depth=[1.0], cov=np.eye(2)[None] * 1e-6, phase=[np.inf])
    with pytest.raises(sdgr.NumericalError, match="primitive 0"):
        sdgr.compute_intensities(sdgr.build_ray_lists(proj), proj)


def test_kat_splat():
    """test_forward.py:191-211: pixel centre, additivity, e^-1 one pixel off."""
    cfg = tiny_config()
    proj = synthetic_projection([[5.0, 7.0]], depth=[1.0], config=cfg)
    buf = sdgr.compute_intensities(sdgr.build_ray_lists(proj), proj)
    img = npa(sdgr.splat_image(buf, proj, cfg))
    assert img[7, 5] == pytest.approx(buf.intensity[0], rel=1e-12)
    assert img[7, 6] == pytest.approx(np.exp(-1.0) * buf.intensity[0], rel=1e-10)
    proj = synthetic_projection([[5.0, 7.0], [5.0, 7.0]], depth=[1.0, 1.0], config=cfg)
    buf = sdgr.compute_intensities(sdgr.build_ray_lists(proj), proj)
    assert npa(sdgr.splat_image(buf, proj, cfg))[7, 5] == pytest.approx(buf.intensity.sum(), rel=1e-12)


def test_kat_splat_permutation_invariance(rng):
    """test_forward.py:213-233 (intensities set directly on the device buffer)."""
    cfg = tiny_config()
    k = 10
    uv = rng.uniform(2, 13, size=(k, 2))
    vals = rng.uniform(0.1, 2.0, k)

    def splat_with(uv_rows, intensity):
        proj = synthetic_projection(uv_rows, depth=np.full(k, 2.0), config=cfg)
        buf = sdgr.compute_intensities(sdgr.build_ray_lists(proj), proj)
        buf.intensity_n.copy_(torch.from_numpy(intensity))
        return npa(sdgr.splat_image(buf, proj, cfg))

    perm = rng.permutation(k)
    np.testing.assert_allclose(splat_with(uv, vals), splat_with(uv[perm], vals[perm]), atol=1e-12)


def test_kat_image_stage():
    """test_backward.py:31-39 (dL/dI = 1) and :49-70 (FD of the splat stage)."""
    cfg = tiny_config()
    proj = synthetic_projection([[5.0, 7.0]], depth=[1.0], config=cfg, cov=np.eye(2)[None] * 1e-6)
    fwd = sdgr.forward_from_projection(proj)
    dl = np.zeros((16, 16))
    dl[7, 5] = 1.0
    dl_di, _, _, _ = sdgr.grad_image_stage(fwd, dl)
    assert dl_di[0] == pytest.approx(1.0, abs=1e-12)

    rng = np.random.default_rng(12345)
    cfg = tiny_config(n=8)
    k = 3
    proj = synthetic_projection(rng.uniform(1, 6, size=(k, 2)), depth=np.arange(k, dtype=float), config=cfg)
    fwd = sdgr.forward_from_projection(proj)
    dl = rng.normal(size=(8, 8))
    dl_di, _, _, _ = sdgr.grad_image_stage(fwd, dl)
    buf, h = fwd.intensities, 1e-5
    for i in range(k):
        orig = float(buf.intensity_n[i])
        buf.intensity_n[i] = orig + h
        up = float(np.sum(dl * npa(sdgr.splat_image(buf, proj, cfg))))
        buf.intensity_n[i] = orig - h
        dn = float(np.sum(dl * npa(sdgr.splat_image(buf, proj, cfg))))
        buf.intensity_n[i] = orig
        assert dl_di[i] == pytest.approx((up - dn) / (2 * h), rel=1e-6, abs=1e-10)


def test_kat_intensity_stage_hand_values():
    """test_backward.py:73-101: dI/dP = 1 - e^-1, dI/dk = e^-1, and a
    shallower Gaussian's extinction attenuates the deeper one."""
    cfg = tiny_config()
    proj = synthetic_projection([[4.0, 4.0]], depth=[1.0], config=cfg, cov=np.eye(2)[None] * 1e-6)
    fwd = sdgr.forward_from_projection(proj)
    dl_dp, dl_dke, _, _ = sdgr.grad_intensity_stage(fwd, np.ones(1))
    assert dl_dp[0] == pytest.approx(1.0 - np.exp(-1.0), abs=1e-9)
    assert dl_dke[0] == pytest.approx(np.exp(-1.0), abs=1e-9)
    cov = np.broadcast_to(np.eye(2) * 1e-6, (2, 2, 2)).copy()
    proj = synthetic_projection([[4.0, 4.0], [4.0, 4.0]], depth=[1.0, 2.0], cov=cov, config=cfg)
    fwd = sdgr.forward_from_projection(proj)
    _, dl_dke, _, _ = sdgr.grad_intensity_stage(fwd, np.array([0.0, 1.0]))
    assert dl_dke[0] < 0.0 and dl_dke[1] > 0.0


def test_synthetic_projection_stages_vs_oracle(rng):
    """Random synthetic projections (anisotropic covariances, varied kappa and
    P) through every device stage against the oracle's stage restatement."""
    k = 20
    uv = rng.uniform(-1.0, 17.0, size=(k, 2))
    cov = np.empty((k, 2, 2))
    for i in range(k):
        a = rng.normal(size=(2, 2))
        cov[i] = a @ a.T + 0.3 * np.eye(2)
    depth, ke, ph = rng.uniform(0, 5, k), rng.uniform(0.1, 3.0, k), rng.uniform(0.2, 2.0, k)
    proj = synthetic_projection(uv, depth, cov=cov, ke_sum=ke, phase=ph)
    fwd = sdgr.forward_from_projection(proj)
    # oracle on the same plane-space inputs
    op = O.OracleProjection(indices=np.arange(k), uv_comp=uv, depth=depth, uv_img=uv, cov_comp=cov, cov_img=cov,
                            phase=ph, phase_unclamped=ph, ke_fwd=ke / 2, ke_bwd=ke / 2,
                            look_dirs=np.tile([0.0, 0.0, 1.0], (k, 1)), look_dists=np.ones(k),
                            view=O.make_view(tiny_config()), n_scene=k, n_culled=0, n_skipped=0, cutoff=3.0)
    rays, spl = O.ray_pairs(op), O.splat_pairs(op)
    inten = O.intensities(rays, op)
    assert np.array_equal(fwd.rays.pair_cell, rays.cell) and np.array_equal(fwd.rays.pair_prim, rays.prim)
    assert_close(fwd.intensities.intensity, inten.intensity, what="intensity")
    assert_close(fwd.image, O.splat(inten.intensity, spl, op), what="image")
    dl = rng.normal(size=(16, 16))
    dI, _, _, _ = sdgr.grad_image_stage(fwd, dl)
    want = np.bincount(spl.prim, weights=dl.reshape(-1)[spl.cell] * spl.w, minlength=k)
    assert_close(dI, want, what="dL/dI")


def test_compositing_exp_accuracy():
    """nexp (the table-driven e^x of the compositing kernels) against
    libdevice exp over the ranges the kernels use (e^-q, q <= 9 + margins;
    e^-S up to the early-stop bound and beyond; underflow, -inf, NaN)."""
    from paper_2506_21633_b200 import _lib

    rng = np.random.default_rng(0)
    x = np.concatenate([-rng.uniform(0, 12, 200000), -rng.uniform(0, 60, 200000), -rng.uniform(0, 800, 50000),
                        -np.logspace(-300, 2.8, 20000), [0.0, -0.0, -1e-320, -707.9, -708.1, -745.0, -746.0,
                                                           -np.inf, np.nan]])
    xd = torch.from_numpy(x).cuda()
    y = torch.empty_like(xd)
    assert _lib.lib().sdgr_exp_check(x.size, xd.data_ptr(), y.data_ptr(), None) == 0
    torch.cuda.synchronize()
    got, ref = y.cpu().numpy(), torch.exp(xd).cpu().numpy()
    fin = np.isfinite(ref) & (ref > 2.3e-308)
    ulp = np.abs(got[fin] - ref[fin]) / np.spacing(ref[fin])
    assert ulp.max() <= 2.0, ulp.max()
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    tiny = ~fin & ~np.isnan(ref)
    assert np.allclose(got[tiny], ref[tiny], rtol=0, atol=1e-307)
