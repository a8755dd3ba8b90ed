"""Profiling driver: one multi-view step of the c4 workload under
cudaProfilerStart/Stop (ncu --profile-from-start off).  Used to produce the
launch lists and ncu captures committed under profiles/."""
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
ap.add_argument("--views", type=int, default=2)
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--size", type=int, default=512)
ap.add_argument("--s-stop", type=float, default=40.0)
a = ap.parse_args()
scene = sdgr.DeviceScene.from_host(bench.make_scene(a.n), dtype=torch.float32)
cfgs = bench.view_list(a.size)[: a.views]
step = MultiViewStep(scene, cfgs, s_stop=a.s_stop)
step.calibrate()
dl = torch.randn((a.views, a.size, a.size), device="cuda", dtype=torch.float64)
step.run(dl)
torch.cuda.synchronize()
torch.cuda.profiler.start()
step.run(dl, check=False)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
step.check()
print("profiled", a.views, "views; launches", sdgr.launch_count())
