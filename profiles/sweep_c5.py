"""BASELINE.json configs[4] / SURVEY.md §8d c5: backward-stress sweep.

c4 layout (16 tanks) with N in {10k, 100k, 1M, 4M} Gaussians and isotropic
scales sigma in {0.03, 0.1, 0.3} m (log_scales overridden), 512x512, el 45°,
8 views per step (one batch).  For each point: member pairs per Gaussian,
(tile, Gaussian) pairs, views/s of forward + backward (CUDA events over a
captured step), and a size-independent check: the step's gradients are
finite and the visible counts equal the number of views that kept each
Gaussian.  Points whose member pairs exceed ~1e9 are skipped.

    python profiles/sweep_c5.py > gpurun_out/c5.json
"""
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200.multiview import MultiViewStep  # noqa: E402

V = 8
cfgs = [c for c in bench.view_list(512) if c.elevation_deg == 45.0][::15][:V]
rows = []
for n in (10_000, 100_000, 1_000_000, 4_000_000):
    base = bench.make_scene(n)
    for sigma in (0.03, 0.1, 0.3):
        est = 9 * math.pi * (sigma ** 2 / 0.09 + 0.3)          # member cells per Gaussian
        if est * n > 1.0e9:
            rows.append({"n": n, "sigma": sigma, "skipped": f"~{est * n:.2e} member pairs"})
            continue
        base.log_scales[:] = math.log(sigma)
        ds = sdgr.DeviceScene.from_host(base, dtype=torch.float32)
        lanes = 8 if est * n < 2e8 else 2
        step = MultiViewStep(ds, cfgs, lanes=lanes)
        step.calibrate()
        dl = torch.randn((V, 512, 512), dtype=torch.float64, device="cuda",
                         generator=torch.Generator("cuda").manual_seed(0))
        step.run(dl)
        step.capture(dl)
        for _ in range(2):
            step.graph_step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            step.graph_step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        step.check()
        g = step.grads
        finite = all(bool(torch.isfinite(getattr(g, k)).all()) for k in
                     ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw", "uv_grad_norm"))
        vis_ok = bool((g.visible >= 0).all() and (g.visible <= V).all())
        rows.append({"n": n, "sigma": sigma, "member_pairs_per_gaussian": float(step.calib_tc) / n,
                     "t16_per_view": step.calib_t16_mean[0], "lanes": lanes, "ms_per_step": ms,
                     "views_per_s": V / (ms / 1e3), "grads_finite": finite, "visible_in_range": vis_ok})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
        del step, ds
        torch.cuda.empty_cache()
print(json.dumps({"config": "c5 backward-stress sweep (BASELINE configs[4])", "views_per_step": V, "rows": rows}))
