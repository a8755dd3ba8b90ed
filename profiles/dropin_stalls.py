"""Where a slow drop-in call spends its time: bench.dropin_rate's call
sequence (c4, 1M Gaussians, 512x512) repeated, each call split into
render_forward / backward, with the events that can stall a call beside it:
result blocks page-locked (scene._OUT_POOL growth), re-binned capacities
(rasterizer._CAPS), caching-allocator device mallocs / retries and host
collections (gc callbacks).

    python profiles/dropin_stalls.py [--profile]
"""
import gc
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_21633_b200 as sdgr  # noqa: E402
from paper_2506_21633_b200 import rasterizer as R, scene as S  # noqa: E402

gc_ms = []
_t = {}


def _gc_cb(phase, info):
    if phase == "start":
        _t["gc"] = time.perf_counter()
    else:
        gc_ms.append((info["generation"], 1e3 * (time.perf_counter() - _t["gc"])))


def main():
    host_scene = bench.make_scene(1_000_000, "c4")
    cfgs = bench.view_list(512, "c4")
    rng = np.random.default_rng(7)
    dls = [rng.normal(size=(512, 512)) for _ in range(10)]
    for i in range(5):
        g = sdgr.backward(sdgr.render_forward(host_scene, cfgs[i % len(cfgs)]), dls[i % 10])
    torch.cuda.synchronize()
    gc.collect()
    gc.callbacks.append(_gc_cb)
    rows = []
    prof = None
    if "--profile" in sys.argv:   # cProfile over the timed calls: the stall's function by tottime
        import cProfile
        prof = cProfile.Profile()
        prof.enable()
    for rep in range(3):
        for i in range(10):
            gc_ms.clear()
            npool = len(S._OUT_POOL)
            caps = dict(R._CAPS)
            m0 = torch.cuda.memory_stats()
            t0 = time.perf_counter()
            fwd = sdgr.render_forward(host_scene, cfgs[i])
            t1 = time.perf_counter()
            g = sdgr.backward(fwd, dls[i])
            t2 = time.perf_counter()
            m1 = torch.cuda.memory_stats()
            rows.append({"rep": rep, "i": i, "fwd_ms": round(1e3 * (t1 - t0), 2), "bwd_ms": round(1e3 * (t2 - t1), 2),
                         "new_blocks": len(S._OUT_POOL) - npool, "recapped": R._CAPS != caps,
                         "dev_mallocs": m1.get("segment.all.allocated", 0) - m0.get("segment.all.allocated", 0),
                         "alloc_retries": m1.get("num_alloc_retries", 0) - m0.get("num_alloc_retries", 0),
                         "gc": [(gen, round(ms, 1)) for gen, ms in gc_ms]})
    del g
    if prof is not None:
        import pstats
        prof.disable()
        pstats.Stats(prof).sort_stats("tottime").print_stats(12)
    for r in rows:
        print(json.dumps(r))
    tot = [r["fwd_ms"] + r["bwd_ms"] for r in rows]
    print(json.dumps({"calls": len(tot), "median_ms": float(np.median(tot)), "max_ms": max(tot),
                      "slow_calls": sum(t > 20 for t in tot)}))


if __name__ == "__main__":
    main()
