"""Synthetic scatterer scenes for parity fixtures and the benchmark.

Mirrors the generators of sarsplat.targets (targets.py:24-223) and the random
scenes of gradcheck.random_scene (gradcheck.py:44-56) draw-for-draw: the same
numpy Generator calls in the same order, so a given seed produces the
reference's exact scene (pinned by tests/test_targets_port.py against
tests/golden/).  Not on the hot path; used to build inputs.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .scene import Scene

SH_C0 = 0.28209479177387814
FACES = ("x-", "x+", "y-", "y+", "z-", "z+")


@dataclass(frozen=True)
class CuboidSpec:
    """Axis-aligned cuboid, base-centered (targets.py:24-59)."""

    height: float
    width: float
    length: float
    center: tuple = (0.0, 0.0, 0.0)
    phase_roof: float = 0.8
    phase_wall: float = 1.0
    extinction: float = 4.0

    @property
    def bounds(self):
        c = np.asarray(self.center, dtype=np.float64)
        lo = c + np.array([-self.width / 2.0, -self.length / 2.0, 0.0])
        hi = c + np.array([self.width / 2.0, self.length / 2.0, self.height])
        return lo, hi

    def face_area(self, face: str) -> float:
        w, l, h = self.width, self.length, self.height
        return {"x-": l * h, "x+": l * h, "y-": w * h, "y+": w * h, "z-": w * l, "z+": w * l}[face]

    def shifted(self, dx: float, dy: float) -> "CuboidSpec":
        c = self.center
        return CuboidSpec(self.height, self.width, self.length, (c[0] + dx, c[1] + dy, c[2]),
                          self.phase_roof, self.phase_wall, self.extinction)


def _face_points(spec: CuboidSpec, face: str, n: int, rng) -> np.ndarray:
    lo, hi = spec.bounds
    u = rng.uniform(size=(n, 2))
    pts = np.empty((n, 3))
    ax = "xyz".index(face[0])
    o1, o2 = [a for a in range(3) if a != ax]
    pts[:, o1] = lo[o1] + u[:, 0] * (hi[o1] - lo[o1])
    pts[:, o2] = lo[o2] + u[:, 1] * (hi[o2] - lo[o2])
    pts[:, ax] = lo[ax] if face[1] == "-" else hi[ax]
    return pts


def sample_cuboid_surface(spec: CuboidSpec, n: int, rng, faces=FACES):
    """Area-weighted surface samples (targets.py:74-94)."""
    if n == 0:
        return np.zeros((0, 3)), np.zeros(0, dtype=np.int64)
    areas = np.array([spec.face_area(f) for f in faces])
    counts = rng.multinomial(n, areas / areas.sum())
    pts = [_face_points(spec, f, c, rng) for f, c in zip(faces, counts)]
    return np.concatenate(pts), np.repeat(np.arange(len(faces)), counts)


def softplus_inverse(y: float) -> float:
    return float(y + np.log(-np.expm1(-y)))      # scene.py:28-33


def _scatterers(points, spacing, phase_dc, extinction) -> Scene:
    """targets.py:121-140."""
    n = points.shape[0]
    sh = np.zeros((n, 16))
    sh[:, 0] = np.asarray(phase_dc, dtype=np.float64) / SH_C0
    rot = np.zeros((n, 4))
    rot[:, 0] = 1.0
    return Scene(points, rot, np.full((n, 3), np.log(spacing)), sh,
                 np.full((n, 2), softplus_inverse(extinction)))


def concatenate(scenes) -> Scene:
    scenes = [s for s in scenes if len(s)]
    return Scene(*(np.concatenate([getattr(s, g) for s in scenes]) for g in
                   ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")))


def building_scene(spec: CuboidSpec, ground_extent: float, density: float, seed: int = 0,
                   ground_phase: float = 0.05, ground_extinction: float = 0.5) -> Scene:
    """Roof + radar-facing wall + ground patch (targets.py:143-183)."""
    rng = np.random.default_rng(seed)
    spacing = 1.0 / np.sqrt(density)
    n_roof = max(1, round(density * spec.face_area("z+")))
    n_wall = max(1, round(density * spec.face_area("x+")))
    roof, _ = sample_cuboid_surface(spec, n_roof, rng, faces=("z+",))
    wall, _ = sample_cuboid_surface(spec, n_wall, rng, faces=("x+",))
    lo, hi = spec.bounds
    half = ground_extent / 2.0
    n_ground = round(density * ground_extent * ground_extent)
    g = rng.uniform(-half, half, size=(n_ground, 2))
    inside = (g[:, 0] > lo[0]) & (g[:, 0] < hi[0]) & (g[:, 1] > lo[1]) & (g[:, 1] < hi[1])
    g = g[~inside]
    ground = np.column_stack([g, np.zeros(len(g))])
    return concatenate([
        _scatterers(roof, spacing, spec.phase_roof, spec.extinction),
        _scatterers(wall, spacing, spec.phase_wall, spec.extinction),
        _scatterers(ground, spacing, ground_phase, ground_extinction),
    ])


def composite_target(specs, n_points, seed: int = 0) -> Scene:
    """Union of sampled cuboids, bottoms excluded (targets.py:186-211)."""
    rng = np.random.default_rng(seed)
    faces = ("x-", "x+", "y-", "y+", "z+")
    parts = []
    for spec, n in zip(list(specs), list(n_points)):
        pts, ids = sample_cuboid_surface(spec, int(n), rng, faces=faces)
        area = sum(spec.face_area(f) for f in faces)
        spacing = np.sqrt(area / max(int(n), 1))
        phase = np.where(ids == faces.index("z+"), spec.phase_roof, spec.phase_wall)
        parts.append(_scatterers(pts, spacing, phase, spec.extinction))
    return concatenate(parts)


def tank_preset(scale: float = 1.0):
    """Hull + turret + barrel (targets.py:214-223)."""
    return [
        CuboidSpec(1.6 * scale, 3.6 * scale, 6.8 * scale, (0.0, 0.0, 0.0), 0.7, 1.0),
        CuboidSpec(0.9 * scale, 2.2 * scale, 3.0 * scale, (0.0, -0.4 * scale, 1.6 * scale), 0.8, 1.1),
        CuboidSpec(0.35 * scale, 0.35 * scale, 3.4 * scale, (0.0, 2.6 * scale, 2.1 * scale), 0.9, 0.9),
    ]


def tank_grid(n_total: int = 1_000_000, grid: int = 4, pitch: float = 20.0, seed: int = 3) -> Scene:
    """tank_preset() translated on a grid x grid lattice
    (pitch m between CuboidSpec centres), per-tank budgets 0.6/0.3/0.1."""
    specs, budgets = [], []
    per = n_total // (grid * grid)
    shares = [int(round(per * 0.6)), int(round(per * 0.3))]
    shares.append(per - shares[0] - shares[1])
    offs = (np.arange(grid) - (grid - 1) / 2.0) * pitch
    for gy in offs:
        for gx in offs:
            for spec, b in zip(tank_preset(), shares):
                specs.append(spec.shifted(float(gx), float(gy)))
                budgets.append(b)
    budgets[-1] += n_total - sum(budgets)
    return composite_target(specs, budgets, seed=seed)


def random_scene(rng, n: int, spread: float = 2.5, dc_low: float = 1.0, dc_high: float = 3.0,
                 scale_low: float = 0.3, scale_high: float = 1.0) -> Scene:
    """gradcheck.random_scene (gradcheck.py:44-56) / tests/conftest.py:23-35."""
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    sh = rng.normal(scale=0.1, size=(n, 16))
    sh[:, 0] = rng.uniform(dc_low, dc_high, size=n)
    return Scene(rng.uniform(-spread, spread, size=(n, 3)), q,
                 rng.uniform(np.log(scale_low), np.log(scale_high), size=(n, 3)), sh,
                 rng.uniform(-0.5, 1.0, size=(n, 2)))


def perturbed(scene: Scene, seed: int = 1) -> Scene:
    """random unit quaternions, log-scales U(log .02, log .3),
    SH DC U(1,3) + N(0, .1) rest, ke_raw U(-.5, 1)."""
    n = len(scene)
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    ls = rng.uniform(np.log(0.02), np.log(0.3), size=(n, 3))
    sh = rng.normal(scale=0.1, size=(n, 16))
    sh[:, 0] = rng.uniform(1.0, 3.0, size=n)
    ke = rng.uniform(-0.5, 1.0, size=(n, 2))
    return Scene(scene.positions.copy(), q, ls, sh, ke)


def to_float32_exact(scene: Scene) -> Scene:
    """Round every parameter to float32 (and back), so float32 and float64
    device scenes describe the same Gaussians bit-for-bit."""
    return Scene(*(getattr(scene, g).astype(np.float32).astype(np.float64)
                   for g in ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")))
