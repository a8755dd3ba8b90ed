"""CPU oracle for the point-cloud evaluation row.

TEST INFRASTRUCTURE ONLY: tests/ use it as the checker of
paper_2506_21633_b200.evaluate; the product never imports it.

Brute-force restatement of the reference's metrics (sarsplat/metrics.py):
  chamfer              metrics.py:140-151  (cKDTree query -> exact nearest neighbour)
  precision_recall_f1  metrics.py:154-162
  dbscan_labels        metrics.py:165-177  (sklearn DBSCAN: radius neighbours with
                       <= eps, itself included; clusters discovered in index order,
                       expanded depth-first from core points, border points keep
                       the first cluster that reaches them)
Pinned against the reference's own outputs in tests/golden/eval/ (made by
tests/golden/make_golden_eval.py with scipy's cKDTree and sklearn's DBSCAN).
"""
from __future__ import annotations

import numpy as np


def _sqdist(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    d = a[:, None, :] - b[None, :, :]
    return np.einsum("ijk,ijk->ij", d, d)


def nn_sqdist(query: np.ndarray, ref: np.ndarray, block: int = 2048) -> np.ndarray:
    out = np.empty(len(query))
    for s in range(0, len(query), block):
        out[s:s + block] = _sqdist(query[s:s + block], ref).min(axis=1)
    return out


def chamfer(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    d_ab = float(np.mean(nn_sqdist(a, b)))
    d_ba = float(np.mean(nn_sqdist(b, a)))
    return d_ab, d_ba, 0.5 * (d_ab + d_ba)


def precision_recall_f1(pred, ref, tau):
    pred, ref = np.asarray(pred, np.float64), np.asarray(ref, np.float64)
    p = float(np.mean(np.sqrt(nn_sqdist(pred, ref)) <= tau))
    r = float(np.mean(np.sqrt(nn_sqdist(ref, pred)) <= tau))
    f1 = 0.0 if p + r == 0 else 2.0 * p * r / (p + r)
    return p, r, f1


def dbscan_labels(points, eps, min_pts):
    pts = np.asarray(points, np.float64)
    n = len(pts)
    nb = [np.flatnonzero(_sqdist(pts[i:i + 1], pts)[0] <= eps * eps) for i in range(n)]
    core = np.array([len(x) >= min_pts for x in nb], dtype=bool)
    labels = np.full(n, -1, dtype=np.int64)
    k = 0
    for i in range(n):
        if labels[i] != -1 or not core[i]:
            continue
        stack = [i]
        labels[i] = k
        while stack:
            j = stack.pop()
            if not core[j]:
                continue
            for m in nb[j]:
                if labels[m] == -1:
                    labels[m] = k
                    stack.append(m)
        k += 1
    return labels
