"""The reference's independent oracles, run through the device drop-in
(B200 only): acceptance criteria 1 and 2 (tests/test_acceptance.py:57-95).

* Criterion 1 (gradient fidelity, gradcheck.py:77-126): the device's
  analytic gradients of L = sum(S^2)/2 (render_forward + backward with
  dL/dS = S, cutoff = inf) against central finite differences of the
  DEVICE render, per group max relative error < 1e-4, clamp-adjacent
  Gaussians excluded as the reference does.
* Criterion 2 (oracle equivalence, forward.py:288-327): device render with
  cutoff = inf against the naive loop renderer (oracle/sdgr_oracle.py
  render_reference, a restatement of the reference's), <= 1e-10 relative.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200 import targets  # noqa: E402
from oracle import sdgr_oracle as O  # noqa: E402

GROUP_SIZES = (("positions", 3), ("rotations", 4), ("log_scales", 3), ("sh_coeffs", 16), ("ke_raw", 2))


def gradcheck_config(rng, size=16):
    """gradcheck.py:59-69."""
    return sdgr.RadarConfig(azimuth_deg=float(rng.uniform(0.0, 360.0)), elevation_deg=float(rng.uniform(38.0, 52.0)),
                            altitude_m=float(rng.uniform(1.0, 4.0)), range_res_m=0.5, azimuth_res_m=0.5,
                            n_range=size, n_azimuth=size)


def gradcheck_scene(rng, n):
    """gradcheck.random_scene (gradcheck.py:44-56): log-scales U(log .3, log 1)."""
    return targets.random_scene(rng, n, scale_low=0.3, scale_high=1.0)


def pack(scene):
    return np.concatenate([getattr(scene, g).ravel() for g, _ in GROUP_SIZES])


def unpack(vec, n):
    parts, o = {}, 0
    for g, w in GROUP_SIZES:
        parts[g] = vec[o:o + n * w].reshape(n, w).copy()
        o += n * w
    return sdgr.Scene(**parts)


def loss(scene, cfg):
    img = sdgr.render(scene, cfg, cutoff=math.inf)
    return 0.5 * float(np.sum(img * img))


def compare_gradients(scene, cfg, step=1e-4):
    """gradcheck.compare_gradients (gradcheck.py:113-126) on the device path."""
    fwd = sdgr.render_forward(scene, cfg, cutoff=math.inf)
    g = sdgr.backward(fwd, fwd.image.copy())
    ana = np.concatenate([a.ravel() for a in g.param_arrays()])
    theta, n = pack(scene), len(scene)
    num = np.empty_like(theta)
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += step
        tm[i] -= step
        num[i] = (loss(unpack(tp, n), cfg) - loss(unpack(tm, n), cfg)) / (2.0 * step)
    proj = sdgr.project_all(scene, cfg, cutoff=math.inf)
    near = np.zeros(n, dtype=bool)
    near[proj.indices] = np.abs(proj.phase_unclamped) < 1e-3
    mask = []
    for grp, w in GROUP_SIZES:
        m = np.ones((n, w), dtype=bool)
        if grp in ("positions", "sh_coeffs"):
            m[near] = False
        mask.append(m.ravel())
    include = np.concatenate(mask)
    denom = np.maximum(np.maximum(np.abs(ana), np.abs(num)), 1e-8)
    rel = np.where(include, np.abs(ana - num) / denom, 0.0)
    out, o = {}, 0
    for grp, w in GROUP_SIZES:
        out[grp] = float(rel[o:o + n * w].max())
        o += n * w
    return out


def test_criterion_1_gradient_fidelity_through_device():
    rng = np.random.default_rng(42)
    worst = {}
    for _ in range(8):
        n = int(rng.integers(3, 11))
        for grp, err in compare_gradients(gradcheck_scene(rng, n), gradcheck_config(rng)).items():
            worst[grp] = max(worst.get(grp, 0.0), err)
    for grp, err in worst.items():
        assert err < 1e-4, f"{grp}: {err:.3e}"


def test_criterion_2_naive_oracle_equivalence_through_device():
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(30):
        n = int(rng.integers(3, 16))
        scene = targets.random_scene(rng, n)
        cfg = gradcheck_config(rng)
        fast = sdgr.render(scene, cfg, cutoff=math.inf)
        slow = O.render_reference(scene, cfg)
        worst = max(worst, np.abs(fast - slow).max() / max(1.0, float(fast.max())))
    assert worst <= 1e-10, worst
