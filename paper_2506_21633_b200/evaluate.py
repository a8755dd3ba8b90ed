"""Point-cloud evaluation on the device.

Same names, arguments, return values and errors as the reference's
``sarsplat.metrics`` (metrics.py:140-183, 206-263): ``chamfer``,
``precision_recall_f1``, ``dbscan_inlier_mask``, ``dbscan_filter``,
``evaluate_point_clouds`` / ``CloudMetricsReport``.  The nearest-neighbour
queries (the reference's cKDTree) and DBSCAN (the reference's sklearn call)
run as libsdgr grid kernels (``sdgr_nn_sqdist``, ``sdgr_dbscan``); torch only
holds the device arrays and does the final means / label compaction.
Points may be numpy arrays or torch tensors of shape (N, 3).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Any

import numpy as np
import torch

from . import _lib
from ._lib import ptr
from .errors import InvalidParameterError

_MAX_DIM_NN = 160        # cells per axis for the NN grid (<= 4.1M cells)
_MAX_DIM_DB = 250        # cells per axis for DBSCAN (<= 15.6M cells)


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2506_21633_b200.evaluate needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _check_points(points, name: str, allow_empty: bool = False) -> torch.Tensor:
    """validation.check_points (validation.py:75-86) on a device FP64 copy."""
    if isinstance(points, torch.Tensor):
        t = points.detach().to(device=_device(), dtype=torch.float64)
    else:
        arr = np.asarray(points, dtype=np.float64)
        if arr.ndim == 1 and arr.size == 0:
            arr = arr.reshape(0, 3)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to(_device())
    if t.ndim == 1 and t.numel() == 0:
        t = t.reshape(0, 3)
    if t.ndim != 2 or t.shape[1] != 3:
        raise InvalidParameterError(f"{name} must have shape (N, 3), got {tuple(t.shape)}")
    if not allow_empty and t.shape[0] == 0:
        raise InvalidParameterError(f"{name} is empty")
    if t.shape[0] and not bool(torch.isfinite(t).all()):
        raise InvalidParameterError(f"{name} contains non-finite coordinates")
    return t.contiguous()


def _check_positive(value, name: str) -> float:
    value = float(value)
    if not np.isfinite(value) or value <= 0:
        raise InvalidParameterError(f"{name} must be a positive finite number, got {value}")
    return value


def _grid(pts: torch.Tensor, h_min: float, max_dim: int, per_cell: float):
    """Corner, cell edge and dims covering pts: edge >= h_min, about
    `per_cell` points per cell, at most `max_dim` cells per axis."""
    lo_t, hi_t = torch.aminmax(pts, dim=0)
    lo, hi = lo_t.cpu().numpy().astype(np.float64), hi_t.cpu().numpy().astype(np.float64)
    ext = np.maximum(hi - lo, 0.0)
    scale = max(float(ext.max()), 1.0)
    vol = float(np.prod(np.maximum(ext, scale * 1e-3)))
    h = max(h_min, (vol * per_cell / max(pts.shape[0], 1)) ** (1.0 / 3.0), float(ext.max()) / (max_dim - 1),
            scale * 1e-9)
    dims = np.minimum(np.floor(ext / h).astype(np.int64) + 1, max_dim).astype(np.int32)
    return (C.c_double * 3)(*lo), h, (C.c_int32 * 3)(*dims), int(np.prod(dims.astype(np.int64)))


def nn_sqdist(query, ref) -> torch.Tensor:
    """Squared distance from every query point to its nearest ref point
    (the cKDTree(ref).query(query)[0] ** 2 of metrics.py:150-160), FP64."""
    q = _check_points(query, "query", allow_empty=True)
    r = _check_points(ref, "ref")
    lib = _lib.lib()
    lo, h, dims, cells = _grid(r, 0.0, _MAX_DIM_NN, 2.0)
    ws_bytes = lib.sdgr_grid_workspace_bytes(r.shape[0], cells)
    ws = torch.empty((ws_bytes,), dtype=torch.uint8, device=r.device)
    out = torch.empty((q.shape[0],), dtype=torch.float64, device=r.device)
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.sdgr_nn_sqdist(ptr(r), r.shape[0], ptr(q), q.shape[0], lo, h, dims, ptr(out), ptr(ws), ws_bytes, st)
    if rc != 0:
        raise RuntimeError(f"sdgr_nn_sqdist: {lib.sdgr_status_string(rc).decode()}")
    return out


def chamfer(a, b):
    """Directed and symmetric Chamfer distances with squared-distance
    averaging (metrics.py:140-151): (d_ab, d_ba, (d_ab + d_ba) / 2)."""
    a = _check_points(a, "a")
    b = _check_points(b, "b")
    d_ab = float(nn_sqdist(a, b).mean().item())
    d_ba = float(nn_sqdist(b, a).mean().item())
    return d_ab, d_ba, 0.5 * (d_ab + d_ba)


def precision_recall_f1(pred, ref, tau: float):
    """Point-matching precision / recall / F1 at distance tolerance tau
    (metrics.py:154-162): a point matches when its nearest-neighbour distance
    in the other set is <= tau."""
    pred = _check_points(pred, "pred")
    ref = _check_points(ref, "ref")
    tau = _check_positive(tau, "tau")
    p = float((torch.sqrt(nn_sqdist(pred, ref)) <= tau).double().mean().item())
    r = float((torch.sqrt(nn_sqdist(ref, pred)) <= tau).double().mean().item())
    f1 = 0.0 if p + r == 0 else 2.0 * p * r / (p + r)
    return p, r, f1


def dbscan_labels(points, eps: float, min_pts: int) -> torch.Tensor:
    """sklearn DBSCAN labels (0..k-1 in the reference's discovery order, -1
    noise) for (N, 3) points, on the device."""
    pts = _check_points(points, "points", allow_empty=True)
    eps = _check_positive(eps, "eps")
    if min_pts < 1:
        raise InvalidParameterError(f"min_pts must be >= 1, got {min_pts}")
    n = pts.shape[0]
    if n == 0:
        return torch.zeros((0,), dtype=torch.int64, device=pts.device)
    lib = _lib.lib()
    lo, h, dims, cells = _grid(pts, eps, _MAX_DIM_DB, 0.0)
    ws_bytes = lib.sdgr_grid_workspace_bytes(n, cells)
    ws = torch.empty((ws_bytes,), dtype=torch.uint8, device=pts.device)
    root = torch.empty((n,), dtype=torch.int32, device=pts.device)
    st = torch.cuda.current_stream().cuda_stream
    rc = lib.sdgr_dbscan(ptr(pts), n, lo, h, dims, eps, int(min_pts), ptr(root), ptr(ws), ws_bytes, st)
    if rc != 0:
        raise RuntimeError(f"sdgr_dbscan: {lib.sdgr_status_string(rc).decode()}")
    # clusters are numbered in order of their smallest core index (sklearn's
    # index-order discovery): dense rank of the roots
    root = root.to(torch.int64)
    labels = torch.full_like(root, -1)
    inl = root >= 0
    if bool(inl.any()):
        uniq = torch.unique(root[inl])      # sorted
        labels[inl] = torch.searchsorted(uniq, root[inl])
    return labels


def dbscan_inlier_mask(points, eps: float, min_pts: int, keep_largest: bool = False) -> np.ndarray:
    """Boolean mask of points belonging to DBSCAN clusters (noise removed),
    optionally only the largest cluster (metrics.py:165-177)."""
    labels = dbscan_labels(points, eps, min_pts)
    if labels.numel() == 0:
        return np.zeros(0, dtype=bool)
    if keep_largest and bool((labels >= 0).any()):
        counts = torch.bincount(labels[labels >= 0])
        return (labels == int(torch.argmax(counts).item())).cpu().numpy()
    return (labels >= 0).cpu().numpy()


def dbscan_filter(points, eps: float, min_pts: int, keep_largest: bool = False) -> np.ndarray:
    """Points with DBSCAN noise removed (metrics.py:180-183)."""
    pts = _check_points(points, "points", allow_empty=True)
    mask = dbscan_inlier_mask(pts, eps, min_pts, keep_largest=keep_largest)
    return pts.cpu().numpy()[mask]


@dataclass
class CloudMetricsReport:
    """Point-cloud reconstruction numbers at a given tolerance (metrics.py:206-230)."""

    dist_ref_to_rec: float
    dist_rec_to_ref: float
    chamfer: float
    precision: float
    recall: float
    f1: float
    tau: float
    extras: dict[str, Any] = field(default_factory=dict)

    def to_record(self) -> dict[str, Any]:
        rec = {"dist_ref_to_rec": self.dist_ref_to_rec, "dist_rec_to_ref": self.dist_rec_to_ref,
               "chamfer": self.chamfer, "precision": self.precision, "recall": self.recall, "f1": self.f1,
               "tau": self.tau}
        rec.update(self.extras)
        return rec


def evaluate_point_clouds(rec, ref, tau: float = 0.6) -> CloudMetricsReport:
    """Chamfer (squared convention) and precision / recall / F1 of rec vs ref
    (metrics.py:251-263)."""
    d_ref_rec, d_rec_ref, cd = chamfer(ref, rec)
    p, r, f1 = precision_recall_f1(rec, ref, tau)
    return CloudMetricsReport(dist_ref_to_rec=d_ref_rec, dist_rec_to_ref=d_rec_ref, chamfer=cd, precision=p,
                              recall=r, f1=f1, tau=tau)


__all__ = ["nn_sqdist", "chamfer", "precision_recall_f1", "dbscan_labels", "dbscan_inlier_mask", "dbscan_filter",
           "CloudMetricsReport", "evaluate_point_clouds"]
