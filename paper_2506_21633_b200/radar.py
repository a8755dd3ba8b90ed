"""Radar view configuration and the per-view constants the kernels consume.

``RadarConfig`` mirrors sarsplat.radar.RadarConfig (radar.py:12-79) field for
field; any object with the same attributes (e.g. the reference's own config)
is accepted wherever a config is expected.

``view_constants`` evaluates, in FP64 on the host, exactly the expressions
the reference evaluates per view (geometry.py:35-128) -- same numpy calls in
the same order -- so the constants handed to the device are bit-identical to
the reference's.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .errors import InvalidParameterError


@dataclass(frozen=True)
class RadarConfig:
    """One side-looking radar view (see sarsplat/radar.py:12-53)."""

    azimuth_deg: float
    elevation_deg: float
    altitude_m: float = 10000.0
    range_res_m: float = 0.3
    azimuth_res_m: float = 0.3
    n_range: int = 128
    n_azimuth: int = 128
    ray_grid: tuple | None = None

    def __post_init__(self):
        if not (0.0 < self.elevation_deg < 90.0):
            raise InvalidParameterError(f"elevation_deg must lie in (0, 90), got {self.elevation_deg}")
        if self.range_res_m <= 0 or self.azimuth_res_m <= 0:
            raise InvalidParameterError("resolutions must be positive")
        if self.n_range < 1 or self.n_azimuth < 1:
            raise InvalidParameterError("image dimensions must be >= 1")
        if self.ray_grid is not None:
            n, m = self.ray_grid
            if n < 1 or m < 1:
                raise InvalidParameterError("ray_grid dimensions must be >= 1")
            object.__setattr__(self, "ray_grid", (int(n), int(m)))
        for name in ("azimuth_deg", "elevation_deg", "altitude_m"):
            if not np.isfinite(getattr(self, name)):
                raise InvalidParameterError(f"{name} must be finite")

    @property
    def n_rays(self) -> tuple:
        return self.ray_grid if self.ray_grid is not None else (self.n_azimuth, self.n_range)

    @property
    def azimuth_rad(self) -> float:
        return float(np.deg2rad(self.azimuth_deg))

    @property
    def elevation_rad(self) -> float:
        return float(np.deg2rad(self.elevation_deg))

    @property
    def slant_range_m(self) -> float:
        return self.altitude_m / np.sin(self.elevation_rad)

    @property
    def ground_extent_m(self) -> float:
        return self.range_res_m * self.n_range

    def with_view(self, azimuth_deg: float, elevation_deg: float) -> "RadarConfig":
        return replace(self, azimuth_deg=azimuth_deg, elevation_deg=elevation_deg)


def n_rays(config) -> tuple:
    rg = getattr(config, "ray_grid", None)
    return tuple(rg) if rg is not None else (config.n_azimuth, config.n_range)


def radar_rotation(azimuth_deg: float, elevation_deg: float) -> np.ndarray:
    """World -> radar rotation (geometry.py:35-47)."""
    phi = np.deg2rad(azimuth_deg)
    theta = np.deg2rad(elevation_deg)
    sp, cp = np.sin(phi), np.cos(phi)
    st, ct = np.sin(theta), np.cos(theta)
    return np.array([[-sp, -cp, 0.0], [-st * cp, st * sp, ct], [-ct * cp, ct * sp, -st]])


def radar_position(config) -> np.ndarray:
    """Platform position (geometry.py:50-56)."""
    phi = float(np.deg2rad(config.azimuth_deg))
    theta = float(np.deg2rad(config.elevation_deg))
    s = config.altitude_m / np.sin(theta)
    return s * np.array([np.cos(theta) * np.cos(phi), -np.cos(theta) * np.sin(phi), np.sin(theta)])


def view_constants(config, cov_reg: float = 0.3, cutoff: float = 3.0) -> _lib.View:
    """Fill the sdgr_view POD for one view (geometry.py:35-128)."""
    R = radar_rotation(config.azimuth_deg, config.elevation_deg)
    cam = radar_position(config)
    T = -R @ cam
    theta = float(np.deg2rad(config.elevation_deg))
    tan_t, sin_t = np.tan(theta), np.sin(theta)
    n_u, n_v = n_rays(config)
    jac_comp = np.array([[n_u / (config.azimuth_res_m * config.n_azimuth), 0.0, 0.0],
                         [0.0, n_v / (config.range_res_m * config.n_range * tan_t), 0.0]])
    jac_img = np.array([[1.0 / config.azimuth_res_m, 0.0, 0.0],
                        [0.0, 0.0, 1.0 / (config.range_res_m * tan_t)]])
    mc = jac_comp @ R
    mi = jac_img @ R
    dr_nr = config.range_res_m * config.n_range
    v = _lib.View()
    v.R[:] = [float(x) for x in R.ravel()]
    v.T[:] = [float(x) for x in T]
    v.cam[:] = [float(x) for x in cam]
    v.mc[:] = [float(x) for x in mc.ravel()]
    v.mi[:] = [float(x) for x in mi.ravel()]
    v.den_u = float(config.azimuth_res_m * config.n_azimuth)
    v.den_v = float(config.range_res_m * config.n_range * tan_t)
    v.off_vi = float(2.0 * config.altitude_m / (dr_nr * sin_t))
    v.cov_reg = float(cov_reg)
    v.cutoff = float(cutoff)
    v.n_u, v.n_v = int(n_u), int(n_v)
    v.n_az, v.n_rg = int(config.n_azimuth), int(config.n_range)
    for d in (v.n_u, v.n_v, v.n_az, v.n_rg):
        if d > 32767:
            raise InvalidParameterError("plane dimensions above 32767 are not supported")
    if np.isnan(cutoff) or cutoff < 0:
        raise InvalidParameterError("cutoff must be >= 0 (or +inf)")
    return v


def view_matrices(config):
    """(R, cam, mc, mi) as numpy arrays, for host-side checks and tests."""
    v = view_constants(config)
    return (np.array(v.R).reshape(3, 3), np.array(v.cam), np.array(v.mc).reshape(2, 3),
            np.array(v.mi).reshape(2, 3))
