"""cProfile of the reference-shaped drop-in call (c2): where the host time goes.

    python profiles/dropin_cprofile.py [c2|c4] > gpurun_out/dropin_cprof.txt
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_21633_b200 as sdgr  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c2"
W = bench.WORKLOADS[w]
scene = bench.make_scene(W["n"], w)
cfgs = bench.view_list(W["size"], w)
dl = np.random.default_rng(0).normal(size=(W["size"], W["size"]))
for i in range(3):
    sdgr.backward(sdgr.render_forward(scene, cfgs[i]), dl)
torch.cuda.synchronize()
calls = 20
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for i in range(calls):
    sdgr.backward(sdgr.render_forward(scene, cfgs[i % len(cfgs)]), dl)
torch.cuda.synchronize()
pr.disable()
print(f"{w}: {1e3 * (time.perf_counter() - t0) / calls:.2f} ms per call (under cProfile)")
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
