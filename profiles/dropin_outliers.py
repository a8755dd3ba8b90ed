import sys, time, gc
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2506_21633_b200 as sdgr
from paper_2506_21633_b200 import rasterizer as R, scene as S
host_scene = bench.make_scene(1_000_000, 'c4')
cfgs = bench.view_list(512, 'c4')
rng = np.random.default_rng(7)
dls = [rng.normal(size=(512, 512)) for _ in range(10)]
for i in range(5):
    g = sdgr.backward(sdgr.render_forward(host_scene, cfgs[i % len(cfgs)]), dls[i % 10])
torch.cuda.synchronize(); gc.collect()
for mode in ("gc on", "gc off"):
    if mode == "gc off": gc.disable()
    out = []
    for i in range(10):
        tc = time.perf_counter()
        npool = len(S._OUT_POOL); ncaps = dict(R._CAPS)
        fwd = sdgr.render_forward(host_scene, cfgs[i])
        g = sdgr.backward(fwd, dls[i])
        out.append((round(1e3*(time.perf_counter()-tc),1), len(S._OUT_POOL) - npool, R._CAPS != ncaps))
    print(mode, out, flush=True)
    gc.enable()
