"""Generate tests/golden/*.npz by running the REFERENCE implementation itself.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Imports sarsplat from /root/reference/pkg/src (read-only; only available in
the build container, never on the GPU box) and records, for a set of seeded
scenes and views, the reference's own outputs of render_forward + backward:
projection arrays, per-cell ray lists (small cases) or their CSR offsets and
a checksum (large cases), 16x16 tile key lists derived per SURVEY.md §8c,
the image and every gradient column.  The oracle (oracle/sdgr_oracle.py) is
pinned against these files by tests/test_oracle_golden.py, and the CUDA path
is checked against them by tests/test_gpu_parity.py.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parents[1]))

import sarsplat as ss  # noqa: E402
from sarsplat.gradcheck import gradcheck_config, random_scene  # noqa: E402

from oracle.sdgr_oracle import Pairs, tile_lists  # noqa: E402  (derivation helper only)

GROUPS = ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")


def checksum(cell: np.ndarray, prim_idx: np.ndarray) -> np.uint64:
    """Order-sensitive 64-bit checksum of a (cell, scene index) pair list."""
    h = np.uint64(1469598103934665603)
    x = (cell.astype(np.uint64) << np.uint64(32)) ^ prim_idx.astype(np.uint64)
    # vectorised FNV-style fold: weight each pair by its position
    w = (np.arange(x.size, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) | np.uint64(1)
    with np.errstate(over="ignore"):
        return np.uint64(h ^ np.bitwise_xor.reduce(x * w)) if x.size else h


class _ProjShim:
    """Adapts a reference Projection to oracle.tile_lists()."""

    def __init__(self, proj, cfg):
        self.indices = proj.indices
        self.depth = proj.depth
        n_u, n_v = cfg.n_rays

        class V:
            pass
        self.view = V()
        self.view.n_u, self.view.n_v = n_u, n_v
        self.view.n_az, self.view.n_rg = cfg.n_azimuth, cfg.n_range

    def __len__(self):
        return len(self.indices)


def record(name: str, scene, cfg, cutoff=3.0, full_pairs=False, grad_rows=None, seed=0):
    fwd = ss.render_forward(scene, cfg, cutoff=cutoff)
    rng = np.random.default_rng(seed)
    dLdS = rng.normal(size=fwd.image.shape)
    g_n = ss.backward(fwd, dLdS)
    g_s = ss.backward(fwd, fwd.image.copy())
    p = fwd.projection
    out = dict(
        cfg=np.array([cfg.azimuth_deg, cfg.elevation_deg, cfg.altitude_m, cfg.range_res_m,
                      cfg.azimuth_res_m, cfg.n_range, cfg.n_azimuth, cutoff], dtype=np.float64),
        indices=p.indices, uv_comp=p.uv_comp, uv_img=p.uv_img, depth=p.depth,
        cov_comp=p.cov_comp[:, [0, 0, 1], [0, 1, 1]], cov_img=p.cov_img[:, [0, 0, 1], [0, 1, 1]],
        phase=p.phase, ke_sum=p.ke_sum, n_culled=p.n_culled, n_skipped=p.n_skipped,
        intensity=fwd.intensities.intensity, image=fwd.image, dLdS=dLdS,
    )
    for plane, pairs_cell, pairs_prim in ((0, fwd.rays.pair_cell, fwd.rays.pair_prim),
                                          (1, fwd.splat.pair_pixel, fwd.splat.pair_prim)):
        pr = Pairs(pairs_cell, pairs_prim, None, None, None, None, None)
        tt, gi, rg = tile_lists(pr, _ProjShim(p, cfg), plane)
        out[f"tiles{plane}_tile"] = tt.astype(np.int32)
        out[f"tiles{plane}_prim"] = gi.astype(np.int32)
        out[f"tiles{plane}_range"] = rg.astype(np.int32)
        out[f"pairs{plane}_count"] = np.int64(len(pairs_cell))
        out[f"pairs{plane}_checksum"] = checksum(pairs_cell, p.indices[pairs_prim])
        if full_pairs:
            out[f"pairs{plane}_cell"] = pairs_cell.astype(np.int32)
            out[f"pairs{plane}_prim"] = p.indices[pairs_prim].astype(np.int32)
    rows = np.arange(len(scene)) if grad_rows is None else grad_rows
    out["grad_rows"] = rows
    for tag, g in (("n", g_n), ("s", g_s)):
        for k in GROUPS + ("uv_grad_norm",):
            out[f"g{tag}_{k}"] = getattr(g, k)[rows]
        out[f"g{tag}_visible"] = g.visible[rows]
    for k in GROUPS:
        out[f"scene_{k}"] = getattr(scene, k)
    np.savez_compressed(HERE / f"{name}.npz", **out)
    print(f"{name}: N={len(scene)} K={len(p)} T_c={len(fwd.rays)} T_i={len(fwd.splat.pair_prim)} "
          f"T16=({len(out['tiles0_tile'])},{len(out['tiles1_tile'])}) "
          f"size={(HERE / f'{name}.npz').stat().st_size // 1024} KiB")


def main():
    # gradcheck-style small scenes (gradcheck.py:44-69), dense and cut
    rng = np.random.default_rng(0)
    for i in range(3):
        scene = random_scene(rng, 5 + 3 * i)
        cfg = gradcheck_config(rng)
        record(f"small{i}_dense", scene, cfg, cutoff=np.inf, full_pairs=True, seed=i)
        record(f"small{i}_cut", scene, cfg, cutoff=3.0, full_pairs=True, seed=i)
    # c1: building, 1 986 Gaussians, 128x128
    c1 = ss.building_scene(ss.CuboidSpec(height=8, width=8, length=10), ground_extent=36,
                           density=1.45, seed=0)
    record("c1_building", c1, ss.RadarConfig(azimuth_deg=0.0, elevation_deg=45.0, altitude_m=1000.0,
                                             range_res_m=0.3, azimuth_res_m=0.3, n_range=128,
                                             n_azimuth=128))
    # c2-lite: 10k tank at 256^2, two views; perturbed copy at 128^2
    tank = ss.composite_target(ss.tank_preset(), [6000, 3000, 1000], seed=3)
    rows = np.random.default_rng(7).choice(len(tank), 1500, replace=False)
    record("tank10k_az37_el45", tank, ss.RadarConfig(azimuth_deg=37.0, elevation_deg=45.0, altitude_m=0.5,
                                                     n_range=256, n_azimuth=256), grad_rows=rows)
    record("tank10k_az200_el15", tank, ss.RadarConfig(azimuth_deg=200.0, elevation_deg=15.0, altitude_m=0.5,
                                                      n_range=256, n_azimuth=256), grad_rows=rows)
    r = np.random.default_rng(1)
    n = len(tank)
    q = r.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sh = r.normal(scale=0.1, size=(n, 16))
    sh[:, 0] = r.uniform(1.0, 3.0, size=n)
    pert = ss.Scene(positions=tank.positions, rotations=q,
                    log_scales=r.uniform(np.log(0.02), np.log(0.3), size=(n, 3)), sh_coeffs=sh,
                    ke_raw=r.uniform(-0.5, 1.0, size=(n, 2)))
    record("tank10k_perturbed_el30", pert, ss.RadarConfig(azimuth_deg=120.0, elevation_deg=30.0,
                                                          altitude_m=0.5, n_range=128, n_azimuth=128),
           grad_rows=rows)
    # non-square image with a custom ray grid
    record("tank10k_raygrid", tank, ss.RadarConfig(azimuth_deg=75.0, elevation_deg=60.0, altitude_m=0.5,
                                                   n_range=96, n_azimuth=160, ray_grid=(120, 80)),
           grad_rows=rows)


if __name__ == "__main__":
    main()
