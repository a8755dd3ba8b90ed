"""Timing of the point-cloud evaluation row on the GPU
box: device grid kernels (paper_2506_21633_b200.evaluate) vs the reference's
CPU implementation of the same calls (scipy cKDTree queries and sklearn
DBSCAN, which is all sarsplat/metrics.py:140-183 does), same inputs.

    python profiles/eval_bench.py [--n-rec 1000000] [--n-ref 300000]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_21633_b200 import evaluate as ev  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n-rec", type=int, default=1_000_000)
ap.add_argument("--n-ref", type=int, default=300_000)
ap.add_argument("--n-db", type=int, default=300_000)
a = ap.parse_args()
rng = np.random.default_rng(0)
ref = rng.uniform(-10, 10, size=(a.n_ref, 3)) * np.array([1, 1, 0.3])
rec = ref[rng.integers(0, a.n_ref, size=a.n_rec)] + rng.normal(0, 0.05, size=(a.n_rec, 3))
rec_d, ref_d = torch.from_numpy(rec).cuda(), torch.from_numpy(ref).cuda()


def gpu_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3, out


def cpu_time(fn):
    t0 = time.perf_counter()
    out = fn()
    return (time.perf_counter() - t0) * 1e3, out


res = {"n_rec": a.n_rec, "n_ref": a.n_ref, "n_db": a.n_db, "cores": len(os.sched_getaffinity(0))}
res["chamfer_gpu_ms"], cd = gpu_time(lambda: ev.chamfer(ref_d, rec_d))
res["prf1_gpu_ms"], prf = gpu_time(lambda: ev.precision_recall_f1(rec_d, ref_d, 0.6))
res["dbscan_gpu_ms"], mask = gpu_time(lambda: ev.dbscan_inlier_mask(rec_d[: a.n_db], 0.1, 5))
try:
    from scipy.spatial import cKDTree
    from sklearn.cluster import DBSCAN

    def ref_chamfer():
        d_ab = float(np.mean(cKDTree(rec).query(ref, workers=-1)[0] ** 2))
        d_ba = float(np.mean(cKDTree(ref).query(rec, workers=-1)[0] ** 2))
        return d_ab, d_ba, 0.5 * (d_ab + d_ba)
    res["chamfer_cpu_ms"], cd_ref = cpu_time(ref_chamfer)
    res["chamfer_rel_diff"] = abs(cd[2] - cd_ref[2]) / cd_ref[2]
    res["dbscan_cpu_ms"], lab = cpu_time(lambda: DBSCAN(eps=0.1, min_samples=5, n_jobs=-1).fit(rec[: a.n_db]).labels_)
    res["dbscan_mask_equal"] = bool(np.array_equal(lab >= 0, mask))
except ImportError as e:   # pragma: no cover
    res["cpu"] = f"unavailable: {e}"
print(json.dumps(res))
