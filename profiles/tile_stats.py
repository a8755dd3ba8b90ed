"""Distribution of per-tile pair counts on the c4 workload (sizes the
per-tile sort kernels)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200.rasterizer import build_ray_lists  # noqa: E402

scene = sdgr.DeviceScene.from_host(bench.make_scene(1_000_000), dtype=torch.float32)
for cfg in bench.view_list(512)[::9]:
    p = sdgr.project_all(scene, cfg)
    tl = build_ray_lists(p)
    r = tl.tile_range.cpu().numpy()
    c = r[:, 1] - r[:, 0]
    print(f"az {cfg.azimuth_deg:5.1f} el {cfg.elevation_deg:4.1f}: pairs {c.sum()} tiles {len(c)} "
          f"max {c.max()} p99 {np.percentile(c, 99):.0f} >4096: {(c > 4096).sum()} >16384: {(c > 16384).sum()} "
          f"pairs in >4096 tiles: {c[c > 4096].sum()}")
