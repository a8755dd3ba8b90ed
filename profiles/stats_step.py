"""Workload statistics of the c4 step, per view: sorted (tile, Gaussian)
pairs, member (ray, Gaussian) pairs, and the live pairs the forward walk
logged under early termination.  Sizes the algorithmic bytes in DESIGN.md."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200.multiview import MultiViewStep  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=45)
ap.add_argument("--s-stop", type=float, default=40.0)
a = ap.parse_args()
scene = sdgr.DeviceScene.from_host(bench.make_scene(1_000_000), dtype=torch.float32)
cfgs = bench.view_list(512)[: a.views]
step = MultiViewStep(scene, cfgs, s_stop=a.s_stop)
step.calibrate()
dl = torch.randn((a.views, 512, 512), device="cuda", dtype=torch.float64)
step.run(dl)
rows = []
for i, v in enumerate(step.views):
    step._preprocess([v], 0)
    step._view(v, dl[i], 0)
    torch.cuda.synchronize()
    t = step.slot_t[0]
    rows.append((int(step.slot_offsets[0][step.n].item()), int(step.member_pairs[0].item()),
                 int(step.member_pairs[1].item()), int(step.replay.cursor[0].item()), int(t["n_items"][0].item())))
n = len(rows)
mean = [sum(r[k] for r in rows) / n for k in range(5)]
print(f"views {n}: comp pairs {mean[0]:.0f}  comp members {mean[1]:.0f}  img members {mean[2]:.0f}  "
      f"live (logged) {mean[3]:.0f} ({100 * mean[3] / max(mean[1], 1):.1f}% of members)  items {mean[4]:.0f}")
for i, r in enumerate(rows[:6]):
    print("  view", i, r)
