"""Generate tests/golden/eval/*.npz by running the REFERENCE's metrics
(sarsplat.metrics: scipy cKDTree, sklearn DBSCAN) on seeded point clouds.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_eval.py

The oracle (oracle/eval_oracle.py) is pinned to these files by
tests/test_eval_oracle.py and the device path checked against them by
tests/test_gpu_eval.py.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sarsplat.metrics import chamfer, dbscan_inlier_mask, precision_recall_f1  # noqa: E402
from sklearn.cluster import DBSCAN  # noqa: E402

OUT = Path(__file__).resolve().parent / "eval"


def clouds(seed: int):
    rng = np.random.default_rng(seed)
    # a reconstruction-like pair: a noisy, partial copy of a box surface + outliers
    ref = rng.uniform(-3, 3, size=(1500, 3)) * np.array([1.0, 0.6, 0.3])
    rec = np.vstack([ref[rng.permutation(len(ref))[:1100]] + rng.normal(0, 0.08, size=(1100, 3)),
                     rng.uniform(-6, 6, size=(40, 3))])
    return rec, ref


def blobs(seed: int):
    rng = np.random.default_rng(seed)
    return np.vstack([rng.normal(0, 0.2, size=(400, 3)), rng.normal(3, 0.3, size=(300, 3)),
                      rng.normal([0, 4, 0], 0.25, size=(200, 3)), rng.uniform(-10, 10, size=(120, 3))])


def main():
    OUT.mkdir(exist_ok=True)
    for seed in (0, 1):
        rec, ref = clouds(seed)
        d_ab, d_ba, cd = chamfer(ref, rec)
        taus = np.array([0.05, 0.1, 0.3, 0.6])
        prf = np.array([precision_recall_f1(rec, ref, t) for t in taus])
        np.savez_compressed(OUT / f"clouds{seed}.npz", rec=rec, ref=ref, chamfer=np.array([d_ab, d_ba, cd]),
                            taus=taus, prf=prf)
    for seed, eps, mp in ((0, 0.3, 5), (1, 0.5, 4), (2, 0.2, 8)):
        pts = blobs(seed)
        labels = DBSCAN(eps=eps, min_samples=mp).fit(pts).labels_
        np.savez_compressed(OUT / f"blobs{seed}.npz", pts=pts, eps=eps, min_pts=mp, labels=labels,
                            mask=dbscan_inlier_mask(pts, eps, mp),
                            mask_largest=dbscan_inlier_mask(pts, eps, mp, keep_largest=True))
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")))


if __name__ == "__main__":
    main()
