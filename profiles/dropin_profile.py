"""Where the time of one reference-shaped drop-in call goes.

    python profiles/dropin_profile.py [c2|c4] > gpurun_out/dropin_<w>.json

Times render_forward(numpy scene) + backward(fwd, numpy dL/dS) -- one view
per call, as the reference's optimize.train calls them (optimize.py:396-411)
-- phase by phase with a device synchronize around each phase (wall clock;
this is a breakdown, not a bench number), then the whole call without the
phase barriers.
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200 import rasterizer as R  # noqa: E402
from paper_2506_21633_b200.scene import as_device_scene  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c4"
W = bench.WORKLOADS[w]
scene = bench.make_scene(W["n"], w)
cfgs = bench.view_list(W["size"], w)
dl = np.random.default_rng(0).normal(size=(W["size"], W["size"]))


def sync():
    torch.cuda.synchronize()


phases = {}


def tick(name, t0):
    sync()
    t = time.perf_counter()
    phases[name] = phases.get(name, 0.0) + 1e3 * (t - t0)
    return t


for it in range(6):
    cfg = cfgs[it % len(cfgs)]
    if it == 1:
        phases.clear()
    sync()
    t = time.perf_counter()
    ds, host = as_device_scene(scene)
    t = tick("upload scene (pageable H2D, FP64)", t)
    proj = R._project(ds, cfg, 0.3, 3.0, True, host)
    t = tick("K1 project", t)
    rays = R._Binner(proj).run((0,))[0]
    t = tick("depth order + binning", t)
    buf = R.compute_intensities(rays, proj, check=False)
    t = tick("compositing (pass A + walk + reduce)", t)
    img = R._splat(buf, proj)
    t = tick("splat", t)
    ov, bad = R._forward_status(buf, proj, [rays])
    t = tick("status read", t)
    fwd = R.ForwardResult(scene=scene, device_scene=ds, config=cfg, projection=proj, rays=rays, intensities=buf,
                          image_t=img, host=True)
    _ = fwd.image
    t = tick("image D2H", t)
    g = R._as_device_grad(dl, fwd)
    t = tick("dL/dS H2D", t)
    acc = R.image_stage_sums(fwd, g)
    t = tick("grad image", t)
    part = R.intensity_stage_partials(fwd, acc[0])
    t = tick("grad intensity (replay)", t)
    gr = R.geometry_stage_fused(fwd, acc, part)
    t = tick("grad geometry", t)
    gr.to_numpy()
    t = tick("gradients D2H (FP64)", t)

calls = 5
phases = {k: v / calls for k, v in phases.items()}
for it in range(3):   # warm the public path itself (its cached pair capacities differ from the exact ones above)
    fwd = sdgr.render_forward(scene, cfgs[it % len(cfgs)])
    sdgr.backward(fwd, dl)
calls = 10
sync()
t0 = time.perf_counter()
for it in range(calls):
    fwd = sdgr.render_forward(scene, cfgs[it % len(cfgs)])
    sdgr.backward(fwd, dl)
sync()
whole = 1e3 * (time.perf_counter() - t0) / calls
print(json.dumps({"workload": w, "phases_ms": phases, "sum_ms": sum(phases.values()), "call_ms": whole,
                  "views_per_s": 1e3 / whole}, indent=1))

# device time per library kernel of one steady-state call (sdgr_profile_*)
import ctypes as C  # noqa: E402

from paper_2506_21633_b200 import _lib  # noqa: E402

lib = _lib.lib()
lib.sdgr_profile_begin(sum(1 << k for k in _lib.KERNEL_NAMES))
sync()
t0 = time.perf_counter()
fwd = sdgr.render_forward(scene, cfgs[0])
sdgr.backward(fwd, dl)
sync()
wall = 1e3 * (time.perf_counter() - t0)
ms = (C.c_double * _lib.PROFILE_KERNELS)()
cnt = (C.c_int64 * _lib.PROFILE_KERNELS)()
lib.sdgr_profile_end(ms, cnt)
print(json.dumps({"one_call_wall_ms": wall,
                  "kernel_ms": {_lib.KERNEL_NAMES[k]: round(ms[k], 4) for k in _lib.KERNEL_NAMES},
                  "launches": {_lib.KERNEL_NAMES[k]: cnt[k] for k in _lib.KERNEL_NAMES}}, indent=1))
