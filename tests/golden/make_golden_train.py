"""Generate tests/golden/train/*.npz by running the REFERENCE loss / SSIM /
Adam code itself.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_train.py

Imports sarsplat from /root/reference/pkg/src (build container only).  Cases:
loss value + dL/dS for several image shapes (windowed SSIM and the
global-window fallback below 11 px) and SSIM weights; two Adam steps on a
random scene with non-finite gradient entries, with and without the
displacement bound.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "train"
sys.path.insert(0, str(REF))

from sarsplat import optimize  # noqa: E402
from sarsplat.backward import SceneGradients  # noqa: E402
from sarsplat.gradcheck import random_scene  # noqa: E402

GROUPS = optimize.PARAM_GROUPS


def loss_cases():
    rng = np.random.default_rng(11)
    out = {}
    for name, (h, w), lam, mv in (("win_48x40", (48, 40), 0.2, 1.0), ("win_64x64_l1", (64, 64), 0.0, 1.0),
                                  ("win_32x33_ssim", (32, 33), 1.0, 2.0), ("global_9x12", (9, 12), 0.2, 1.0),
                                  ("win_11x11", (11, 11), 0.5, 1.0)):
        S = rng.uniform(0.0, 1.0, size=(h, w))
        Y = np.clip(S + rng.normal(0.0, 0.1, size=(h, w)), 0.0, None)
        S[0, 0] = Y[0, 0]  # a zero difference (sign 0)
        value, grad = optimize.loss(S, Y, lam, max_val=mv)
        out[name] = dict(S=S, Y=Y, lam=np.float64(lam), max_val=np.float64(mv), value=np.float64(value), grad=grad)
    return out


def adam_case(bound):
    rng = np.random.default_rng(5)
    scene = random_scene(rng, 64)
    state = optimize.AdamState.for_scene(scene)
    lrs = {"positions": 1e-2, "rotations": 1e-3, "log_scales": 5e-3, "sh_coeffs": 2.5e-3, "ke_raw": 5e-2}
    rec = {f"p0_{g}": getattr(scene, g).copy() for g in GROUPS}
    for k in range(2):
        gr = {g: rng.normal(0.0, 1.0, size=getattr(scene, g).shape).astype(np.float32).astype(np.float64)
              for g in GROUPS}
        gr["sh_coeffs"][3, 5] = np.nan
        gr["positions"][7, 1] = np.inf
        grads = SceneGradients(gr["positions"], gr["rotations"], gr["log_scales"], gr["sh_coeffs"], gr["ke_raw"],
                               np.zeros(len(scene)), np.ones(len(scene), bool))
        for g in GROUPS:
            rec[f"g{k}_{g}"] = gr[g]
        optimize.adam_step(scene, grads, state, lrs, displacement_bound=bound)
        for g in GROUPS:
            rec[f"p{k + 1}_{g}"] = getattr(scene, g).copy()
            rec[f"m{k + 1}_{g}"] = state.m[g].copy()
            rec[f"v{k + 1}_{g}"] = state.v[g].copy()
    rec["n_skipped"] = np.int64(state.n_skipped)
    rec["lrs"] = np.array([lrs[g] for g in GROUPS])
    rec["bound"] = np.float64(-1.0 if bound is None else bound)
    return rec


def densify_case():
    """densify_and_prune (optimize.py:251-312) with clones, splits and prunes."""
    rng = np.random.default_rng(9)
    scene = random_scene(rng, 300)
    view = optimize.RadarConfig(azimuth_deg=0.0, elevation_deg=45.0, range_res_m=0.3, n_range=64)  # cap 5.76
    scene.log_scales[:20] = np.log(rng.uniform(6.0, 9.0, size=(20, 3)))        # oversized -> split
    scene.log_scales[20:80] = np.log(rng.uniform(0.005, 0.05, size=(60, 3)))   # small -> clone candidates
    scene.sh_coeffs[280:, 0] = 0.001                                           # weak phase -> pruned
    n = len(scene)
    accum = optimize.GradAccumulator.zeros(n)
    accum.norm_sum[:] = rng.uniform(0.0, 0.02, size=n)
    accum.pos_sum[:] = rng.normal(0.0, 1.0, size=(n, 3))
    accum.count[:] = rng.integers(0, 4, size=n).astype(np.float64)
    state = optimize.AdamState.for_scene(scene)
    for g in GROUPS:
        state.m[g][:] = rng.normal(size=state.m[g].shape)
        state.v[g][:] = rng.uniform(size=state.v[g].shape)
    cfg = optimize.TrainConfig()
    rec = {f"in_{g}": getattr(scene, g).copy() for g in GROUPS}
    rec.update({f"in_m_{g}": state.m[g].copy() for g in GROUPS})
    rec.update({f"in_v_{g}": state.v[g].copy() for g in GROUPS})
    rec.update(norm_sum=accum.norm_sum.copy(), pos_sum=accum.pos_sum.copy(), count=accum.count.copy())
    extent, lr, seed = 10.0, 0.02, 7
    out, acc2, ev = optimize.densify_and_prune(scene, accum, cfg, view, extent, lr, np.random.default_rng(seed),
                                               state=state)
    rec.update({f"out_{g}": getattr(out, g) for g in GROUPS})
    rec.update({f"out_m_{g}": state.m[g] for g in GROUPS})
    rec.update({f"out_v_{g}": state.v[g] for g in GROUPS})
    rec.update(event=np.array([ev.n_cloned, ev.n_split, ev.n_pruned, ev.n_after]), extent=np.float64(extent),
               lr=np.float64(lr), seed=np.int64(seed), ground_extent=np.float64(view.ground_extent_m),
               cfg=np.array([cfg.densify_grad_threshold, cfg.max_radius_factor, cfg.clone_size_factor,
                             cfg.prune_phase_floor, cfg.split_scale_shrink]))
    return rec


def main():
    OUT.mkdir(exist_ok=True)
    for name, d in loss_cases().items():
        np.savez_compressed(OUT / f"loss_{name}.npz", **d)
    np.savez_compressed(OUT / "adam_free.npz", **adam_case(None))
    np.savez_compressed(OUT / "adam_bound.npz", **adam_case(0.004))
    np.savez_compressed(OUT / "densify.npz", **densify_case())
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
