import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

GROUPS = ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")
# north-star tolerance (BASELINE.json): |gpu - ref| <= 1e-6 + 1e-4 |ref|
ATOL, RTOL = 1e-6, 1e-4


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsdgr.so")
    config.addinivalue_line("markers", "slow: long-running")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")


def golden_files():
    return sorted(GOLDEN.glob("*.npz"))


def load_golden(path):
    from paper_2506_21633_b200.radar import RadarConfig
    from paper_2506_21633_b200.scene import Scene

    z = np.load(path)
    az, el, alt, dr, da, nr, na, cutoff = z["cfg"]
    name = Path(path).stem
    ray_grid = (120, 80) if "raygrid" in name else None
    cfg = RadarConfig(azimuth_deg=float(az), elevation_deg=float(el), altitude_m=float(alt),
                      range_res_m=float(dr), azimuth_res_m=float(da), n_range=int(nr),
                      n_azimuth=int(na), ray_grid=ray_grid)
    scene = Scene(*(z[f"scene_{g}"] for g in GROUPS))
    return z, scene, cfg, float(cutoff)


def assert_close(got, ref, atol=ATOL, rtol=RTOL, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    bad = np.abs(got - ref) > atol + rtol * np.abs(ref)
    if bad.any():
        i = np.flatnonzero(bad.ravel())[0]
        raise AssertionError(
            f"{what}: {int(bad.sum())}/{bad.size} outside tol; first at {i}: got {got.ravel()[i]!r} "
            f"ref {ref.ravel()[i]!r}; max abs err {np.abs(got - ref).max():.3e}")


def npa(x):
    """numpy view of a reference-shaped result (numpy for host callers,
    a CUDA tensor for device callers)."""
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def has_reference() -> bool:
    return (REFERENCE_SRC / "sarsplat" / "__init__.py").exists()
