"""Concurrency timeline of one captured c4 step (45 views, 8 lanes).

    python profiles/timeline.py > gpurun_out/timeline.json

Every library kernel launch of one graph replay is bracketed by event nodes
(sdgr_profile_begin / sdgr_profile_timeline); the report gives, per kernel,
the summed ready->done spans, and over the step the time with k = 0, 1, 2, ...
launches in flight -- where the concurrent step leaves the GPU idle or runs
one latency-bound kernel alone.
"""
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200 import _lib  # noqa: E402
from paper_2506_21633_b200.multiview import MultiViewStep  # noqa: E402

scene = sdgr.DeviceScene.from_host(bench.make_scene(1_000_000), dtype=torch.float32)
cfgs = bench.view_list(512)[:45]
step = MultiViewStep(scene, cfgs)
step.calibrate()
dl = torch.randn((45, 512, 512), device="cuda", dtype=torch.float64)
for _ in range(3):
    step.run(dl)
lib = _lib.lib()
lib.sdgr_profile_begin(sum(1 << k for k in _lib.KERNEL_NAMES))
step.capture(dl, warm=False)
step.graph_step()
torch.cuda.synchronize()
cap = 4096
ids = (C.c_int32 * cap)()
t0 = (C.c_double * cap)()
t1 = (C.c_double * cap)()
n = lib.sdgr_profile_timeline(cap, ids, t0, t1)
ms = (C.c_double * _lib.PROFILE_KERNELS)()
cnt = (C.c_int64 * _lib.PROFILE_KERNELS)()
lib.sdgr_profile_end(ms, cnt)
ev = [(t0[i], t1[i], _lib.KERNEL_NAMES.get(ids[i], str(ids[i]))) for i in range(n)]
end = max(e[1] for e in ev)
# in-flight histogram over the step
pts = sorted([(a, 1) for a, _, _ in ev] + [(b, -1) for _, b, _ in ev])
hist, cur, last = {}, 0, 0.0
for t, d in pts:
    hist[cur] = hist.get(cur, 0.0) + (t - last)
    cur += d
    last = t
per = {}
for a, b, nm in ev:
    p = per.setdefault(nm, [0, 0.0])
    p[0] += 1
    p[1] += b - a
first_walk = min((a for a, _, nm in ev if nm == "k_walk<kContrib>"), default=None)
# which kernel runs alone during the single-kernel periods
solo = {}
bounds = sorted({x for a, b, _ in ev for x in (a, b)})
for lo, hi in zip(bounds, bounds[1:]):
    live = [nm for a, b, nm in ev if a <= lo and b >= hi]
    if len(live) == 1:
        solo[live[0]] = solo.get(live[0], 0.0) + (hi - lo)
print(json.dumps({"launches": n, "step_span_ms": end,
                  "ms_with_k_in_flight": {str(k): round(v, 3) for k, v in sorted(hist.items())},
                  "first_walk_starts_ms": first_walk,
                  "ready_to_done_ms_per_kernel": {k: round(v[1], 3) for k, v in per.items()},
                  "launch_counts": {k: v[0] for k, v in per.items()},
                  "solo_ms_by_kernel": {k: round(v, 3) for k, v in sorted(solo.items(), key=lambda x: -x[1])},
                  "events": [[round(a, 4), round(b, 4), nm] for a, b, nm in sorted(ev)]}, indent=1))
