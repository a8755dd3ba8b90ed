import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2506_21633_b200 as sdgr
w = sys.argv[1]
W = bench.WORKLOADS[w]
scene = bench.make_scene(W["n"], w)
cfgs = bench.view_list(W["size"], w)
dl = np.random.default_rng(0).normal(size=(W["size"], W["size"]))
for it in range(12):
    torch.cuda.synchronize(); t = time.perf_counter()
    fwd = sdgr.render_forward(scene, cfgs[it % len(cfgs)])
    g = sdgr.backward(fwd, dl)
    torch.cuda.synchronize()
    print(it, round(1e3 * (time.perf_counter() - t), 2), fwd.rays.capacity if hasattr(fwd.rays, 'capacity') else None, flush=True)
