import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_2506_21633_b200.scene import upload_f64, download
import os
print("cpus", len(os.sched_getaffinity(0)))
a = [np.random.rand(1_000_000, w) for w in (3, 4, 3, 16, 2)]
d = [torch.rand(1_000_000, w, dtype=torch.float64, device="cuda") for w in (3, 4, 3, 16, 2)] + [torch.rand(1_000_000, dtype=torch.float64, device="cuda")]
for rep in range(6):
    torch.cuda.synchronize(); t = time.perf_counter()
    for x in a: upload_f64(x, "cuda")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    out = download(d)
    t2 = time.perf_counter()
    for x in a: torch.from_numpy(x).cuda()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    for x in d: x.cpu().numpy()
    t4 = time.perf_counter()
    print(f"up staged {1e3*(t1-t):.1f} ms  down staged {1e3*(t2-t1):.1f} ms  up pageable {1e3*(t3-t2):.1f}  down pageable {1e3*(t4-t3):.1f}")
