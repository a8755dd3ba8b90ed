"""Raw cost of a caching-allocator miss on this box: torch.empty of fresh
device segments (cudaMalloc) of growing size after empty_cache."""
import time
import torch
torch.cuda.init()
x = torch.empty(1, device="cuda")
for mb in (2, 64, 256, 1024, 4096):
    ts = []
    for _ in range(3):
        torch.cuda.synchronize(); torch.cuda.empty_cache()
        t0 = time.perf_counter()
        a = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
        ts.append(round(1e3 * (time.perf_counter() - t0), 2))
        del a
    print(f"{mb} MB: cudaMalloc ms {ts}", flush=True)
