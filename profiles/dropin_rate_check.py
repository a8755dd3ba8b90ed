import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2506_21633_b200 as sdgr
host_scene = bench.make_scene(1_000_000, 'c4')
cfgs = bench.view_list(512, 'c4')
for rep in range(3):
    t = time.perf_counter()
    r = bench.dropin_rate(sdgr, host_scene, cfgs, 6, 1, 0)
    print(rep, round(r['value'], 1), round(r['ms_per_view'], 2), round(time.perf_counter() - t, 2), flush=True)
