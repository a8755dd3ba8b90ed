"""CPU restatement of the training-step pieces around the SDGR path -- TEST
INFRASTRUCTURE ONLY (imported by tests/ as the checker; never by the product).

Follows the reference line by line:
  loss            optimize.py:85-102
  ssim_with_grad  metrics.py:98-137 (_ssim_kernel :45-49, _ssim_filter :52-55,
                  _ssim_terms :58-76)
  adam_step       optimize.py:171-207
  densify_and_prune optimize.py:251-312 (covariances: scene.py:49-97)
Pinned by tests/test_train_oracle.py against tests/golden/train/*.npz, which
tests/golden/make_golden_train.py produced by running the reference itself.
The separable filter is restated with explicit zero padding instead of
scipy.ndimage.correlate1d (same sums, possibly different rounding order).
"""
from __future__ import annotations

import numpy as np

WIN, SIGMA, K1, K2 = 11, 1.5, 0.01, 0.03
GROUPS = ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")


def ssim_kernel():
    # metrics.py:45-49
    r = (WIN - 1) // 2
    t = np.arange(-r, r + 1, dtype=np.float64)
    k = np.exp(-(t * t) / (2.0 * SIGMA * SIGMA))
    return k / k.sum()


def _corr1d(img, k, axis):
    # correlate1d(mode="constant", cval=0): out[i] = sum_t k[t] img[i + t - r]
    r = (len(k) - 1) // 2
    a = np.moveaxis(img, axis, 0)
    pad = np.zeros((a.shape[0] + 2 * r,) + a.shape[1:])
    pad[r:r + a.shape[0]] = a
    out = np.zeros_like(a)
    for t in range(len(k)):
        out += k[t] * pad[t:t + a.shape[0]]
    return np.moveaxis(out, 0, axis)


def _filter(img, k):
    # metrics.py:52-55: axis 0, then axis 1
    return _corr1d(_corr1d(img, k, 0), k, 1)


def _terms(x, y, max_val, k):
    # metrics.py:58-76
    c1 = (K1 * max_val) ** 2
    c2 = (K2 * max_val) ** 2
    if k is None:
        def filt(z):
            return np.full_like(z, z.mean())
    else:
        def filt(z):
            return _filter(z, k)
    ux, uy = filt(x), filt(y)
    ex2, ey2, exy = filt(x * x), filt(y * y), filt(x * y)
    vx, vy = ex2 - ux * ux, ey2 - uy * uy
    cxy = exy - ux * uy
    a1 = 2.0 * ux * uy + c1
    a2 = 2.0 * cxy + c2
    b1 = ux * ux + uy * uy + c1
    b2 = vx + vy + c2
    return filt, ux, uy, a1, a2, b1, b2


def ssim_with_grad(x, y, max_val=1.0):
    # metrics.py:98-137
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    windowed = min(x.shape) >= WIN
    k = ssim_kernel() if windowed else None
    filt, ux, uy, a1, a2, b1, b2 = _terms(x, y, max_val, k)
    denom = b1 * b2
    smap = (a1 * a2) / denom
    weight = np.zeros_like(x)
    if windowed:
        pad = (WIN - 1) // 2
        n_win = (x.shape[0] - 2 * pad) * (x.shape[1] - 2 * pad)
        weight[pad:-pad, pad:-pad] = 1.0 / n_win
        value = float(smap[pad:-pad, pad:-pad].mean())
    else:
        weight[:] = 1.0 / x.size
        n_total = x.size
        value = float(smap.flat[0])
    ds_da1 = a2 / denom
    ds_da2 = a1 / denom
    ds_db1 = -smap / b1
    ds_db2 = -smap / b2
    ds_dux = ds_da1 * 2.0 * uy + ds_da2 * (-2.0 * uy) + ds_db1 * 2.0 * ux + ds_db2 * (-2.0 * ux)
    ds_dex2 = ds_db2
    ds_dexy = ds_da2 * 2.0
    if windowed:
        def back(z):
            return _filter(z, k)
    else:
        def back(z):
            return np.full_like(z, z.sum() / n_total)
    grad = back(weight * ds_dux) + 2.0 * x * back(weight * ds_dex2) + y * back(weight * ds_dexy)
    return value, grad


def loss(rendered, target, lambda_ssim=0.2, max_val=1.0):
    # optimize.py:85-102
    rendered = np.asarray(rendered, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    diff = rendered - target
    l1 = float(np.mean(np.abs(diff)))
    grad = np.sign(diff) / diff.size * (1.0 - lambda_ssim)
    value = (1.0 - lambda_ssim) * l1
    if lambda_ssim > 0.0:
        s, ds = ssim_with_grad(rendered, target, max_val=max_val)
        value += lambda_ssim * (1.0 - s)
        grad -= lambda_ssim * ds
    return value, grad


def adam_step(params, grads, m, v, step, lrs, displacement_bound=None, b1=0.9, b2=0.999, eps=1e-8):
    """optimize.py:171-207 on dicts of float64 arrays (params/m/v updated in
    place); returns (new step, number of zeroed non-finite entries)."""
    step += 1
    bc1 = 1.0 - b1 ** step
    bc2 = 1.0 - b2 ** step
    skipped = 0
    for g in GROUPS:
        grad = grads[g]
        bad = ~np.isfinite(grad)
        if bad.any():
            skipped += int(bad.sum())
            grad = np.where(bad, 0.0, grad)
        mm, vv = m[g], v[g]
        mm *= b1
        mm += (1.0 - b1) * grad
        vv *= b2
        vv += (1.0 - b2) * grad * grad
        st = lrs[g] * (mm / bc1) / (np.sqrt(vv / bc2) + eps)
        if g == "positions" and displacement_bound is not None:
            norms = np.linalg.norm(st, axis=1, keepdims=True)
            factor = np.minimum(1.0, displacement_bound / np.maximum(norms, 1e-300))
            st = st * factor
        params[g] -= st
    params["rotations"] /= np.linalg.norm(params["rotations"], axis=1, keepdims=True)
    return step, skipped


def covariances(rotations, log_scales):
    # scene.py:49-97 (quats_to_rotation_matrices + covariances_from_arrays)
    q = rotations / np.linalg.norm(rotations, axis=-1, keepdims=True)
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((len(q), 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    M = R * np.exp(log_scales)[:, None, :]
    cov = M @ np.swapaxes(M, -1, -2)
    return 0.5 * (cov + np.swapaxes(cov, -1, -2))


SH_C0 = 0.28209479177387814


def densify_and_prune(params, norm_sum, pos_sum, count, cfg, ground_extent, extent, lr, rng, m=None, v=None):
    """optimize.py:251-312 on dicts of float64 arrays.  cfg = (grad_threshold,
    max_radius_factor, clone_size_factor, prune_phase_floor, split_scale_shrink).
    Returns (new params, (n_cloned, n_split, n_pruned, n_after), new m, new v)."""
    thr, radius_factor, clone_factor, floor, shrink = cfg
    cap = radius_factor * ground_extent
    max_scale = np.exp(params["log_scales"]).max(axis=1)
    split = max_scale > cap
    small = max_scale <= clone_factor * extent
    mean_norm = norm_sum / np.maximum(count, 1.0)
    clone = (mean_norm > thr) & small & ~split & (count > 0)
    kept = ~split
    parts = [{g: params[g][kept] for g in GROUPS}]
    n_clone = int(clone.sum())
    if n_clone:
        c = {g: params[g][clone] for g in GROUPS}
        c["positions"] = c["positions"] + (-lr * (pos_sum / np.maximum(count, 1.0)[:, None])[clone])
        parts.append(c)
    n_split = int(split.sum())
    if n_split:
        rows = np.repeat(np.flatnonzero(split), 2)
        ch = {g: params[g][rows] for g in GROUPS}
        chol = np.linalg.cholesky(covariances(ch["rotations"], ch["log_scales"]))
        xi = rng.normal(size=(len(rows), 3))
        ch["positions"] = ch["positions"] + np.einsum("kab,kb->ka", chol, xi)
        ch["log_scales"] = ch["log_scales"] - np.log(shrink)
        parts.append(ch)
    merged = {g: np.concatenate([p[g] for p in parts]) for g in GROUPS}
    dc_phase = merged["sh_coeffs"][:, 0] * SH_C0
    oversized = np.exp(merged["log_scales"]).max(axis=1) > cap
    survive = (dc_phase >= floor) & ~oversized
    out = {g: merged[g][survive] for g in GROUPS}
    new_m = new_v = None
    if m is not None:
        n_new = n_clone + 2 * n_split

        def reidx(d):
            return {g: np.concatenate([d[g][kept], np.zeros((n_new,) + d[g].shape[1:])])[survive] for g in GROUPS}
        new_m, new_v = reidx(m), reidx(v)
    event = (n_clone, n_split, int((~survive).sum()), int(survive.sum()))
    return out, event, new_m, new_v
