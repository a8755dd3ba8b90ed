"""Cycle breakdown of the forward tile walk by phase (profiling build).

    SDGR_LIB_NAME=libsdgr_prof.so SDGR_EXTRA_FLAGS=-DSDGR_WALK_PROFILE SDGR_BUILD_SUFFIX=_prof \\
        python -m paper_2506_21633_b200.csrc.build
    SDGR_LIB=libsdgr_prof.so python profiles/walk_phases.py

Thread 0 of every walk CTA adds the clock64() cycles between the barriers
that close each phase; shares are of the summed CTA time."""
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("SDGR_LIB", "libsdgr_prof.so")

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200 import _lib  # noqa: E402
from paper_2506_21633_b200.multiview import MultiViewStep  # noqa: E402

NAMES = ["item claim / item tail", "P0 record load + member mask", "-", "live test + scatter + ballot",
         "count scan + sub-chunk fit", "P1 ray counts + scan", "P2 weights (exp)", "P3 prefix + replay claim",
         "P4 T, 1-e^-tau, log writes", "P7 per-Gaussian reduce", "P3 prefix (profile barrier)"]
views = int(sys.argv[1]) if len(sys.argv) > 1 else 8
scene = sdgr.DeviceScene.from_host(bench.make_scene(1_000_000), dtype=torch.float32)
step = MultiViewStep(scene, bench.view_list(512)[:views])
step.calibrate()
dl = torch.randn((views, 512, 512), device="cuda", dtype=torch.float64)
step.run(dl)
lib = _lib.lib()
fn = lib.sdgr_debug_walk_profile
fn.argtypes = [C.POINTER(C.c_uint64)]
out = (C.c_uint64 * 16)()
torch.cuda.synchronize()
fn(out)  # reset
step.run(dl)
torch.cuda.synchronize()
fn(out)
tot = sum(out[:11]) or 1
print(f"walk CTA cycles over {views} views (forward + rewalk modes): {tot:.3e}")
for i, nm in enumerate(NAMES):
    if nm != "-":
        print(f"  {i}: {100 * out[i] / tot:5.1f}%  {nm}" + ("  (replay claim wait when 10 is present)" if i == 7 else ""))
