"""Gaussian-scatterer scenes: host mirror and device-resident SoA.

``Scene`` mirrors sarsplat.scene.Scene (scene.py:132-244): five contiguous
float64 arrays.  ``DeviceScene`` holds the same five arrays as CUDA tensors
(float32 or float64), 16-byte aligned, the layout the kernels read.  Every
public entry point accepts either, or any object exposing the five
attributes (e.g. the reference's own Scene).
"""
from __future__ import annotations

import gc
import sys
import threading
import weakref
from dataclasses import dataclass, field
from typing import Any

import numpy as np
import torch

GROUPS = (("positions", 3), ("rotations", 4), ("log_scales", 3), ("sh_coeffs", 16), ("ke_raw", 2))


@dataclass
class Scene:
    """Host-side scene, float64 SoA (scene.py:132-158)."""

    positions: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    sh_coeffs: np.ndarray
    ke_raw: np.ndarray
    metadata: dict[str, Any] = field(default_factory=dict)

    def __post_init__(self):
        n = len(self.positions)
        for name, w in GROUPS:
            setattr(self, name, np.ascontiguousarray(getattr(self, name), dtype=np.float64).reshape(n, w))

    def __len__(self) -> int:
        return self.positions.shape[0]

    def copy(self) -> "Scene":
        return Scene(*(getattr(self, g).copy() for g, _ in GROUPS), metadata=dict(self.metadata))

    @classmethod
    def empty(cls) -> "Scene":
        return cls(*(np.zeros((0, w)) for _, w in GROUPS))


@dataclass
class DeviceScene:
    """Device-resident scene: five (n, w) CUDA tensors of one dtype."""

    positions: torch.Tensor
    rotations: torch.Tensor
    log_scales: torch.Tensor
    sh_coeffs: torch.Tensor
    ke_raw: torch.Tensor

    def __len__(self) -> int:
        return int(self.positions.shape[0])

    @property
    def dtype(self) -> torch.dtype:
        return self.positions.dtype

    @property
    def device(self) -> torch.device:
        return self.positions.device

    def arrays(self):
        return tuple(getattr(self, g) for g, _ in GROUPS)

    @classmethod
    def from_host(cls, scene, dtype=torch.float64, device="cuda", pin: bool = False) -> "DeviceScene":
        """Upload any Scene-like object (numpy or torch fields)."""
        out = []
        for g, w in GROUPS:
            a = getattr(scene, g)
            t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
            t = t.reshape(-1, w).to(dtype)
            if pin and t.device.type == "cpu":
                t = t.pin_memory()
            out.append(t.to(device, non_blocking=True).contiguous())
        return cls(*out)

    def to_host(self) -> Scene:
        return Scene(*(t.detach().double().cpu().numpy() for t in self.arrays()))


def spatial_order(positions) -> np.ndarray:
    """Permutation that puts Gaussians in 3-D Morton (Z-curve) order of their
    positions (10 bits per axis over the bounding box; ties keep their
    original order).  Neighbouring Gaussians then sit next to each other in
    memory: the per-Gaussian kernels (emission, record gather, imaging-plane
    backward, geometry) read and write nearby rows, and a warp's tile pairs
    and pixels overlap.  c4: 1336 -> 1361 views/s against the sampler's own
    order, 1275 for a random order (profiles/ROUND2.md).  Rendering is
    order-independent apart from exact depth ties (the reference breaks
    them by projection row, forward.py:147), so a sorted scene renders the
    same image and its gradients are the original's, permuted (up to the
    rounding of the order-dependent sums)."""
    p = positions.detach().double().cpu().numpy() if isinstance(positions, torch.Tensor) else np.asarray(positions)
    p = p.reshape(-1, 3)
    if len(p) == 0:
        return np.zeros((0,), np.int64)
    lo = np.nanmin(np.where(np.isfinite(p), p, np.nan), axis=0)
    span = np.nanmax(np.where(np.isfinite(p), p, np.nan), axis=0) - lo
    lo, span = np.nan_to_num(lo), np.nan_to_num(span)
    q = np.clip(np.nan_to_num((p - lo) / max(float(span.max()), 1e-300) * 1023.0), 0, 1023).astype(np.int64)
    code = np.zeros(len(p), np.int64)
    for b in range(10):
        for a in range(3):
            code |= ((q[:, a] >> b) & 1) << (3 * b + a)
    return np.argsort(code, kind="stable")


def spatial_sort(scene):
    """(scene in spatial_order, perm): sorted[i] = scene[perm[i]].  Host
    scenes come back as Scene, device scenes as DeviceScene; gradients of
    the sorted scene map back with g_original[perm] = g_sorted."""
    perm = spatial_order(scene.positions)
    if isinstance(scene.positions, torch.Tensor):
        idx = torch.from_numpy(perm).to(scene.positions.device)
        return DeviceScene(*(getattr(scene, g).reshape(-1, w)[idx].contiguous() for g, w in GROUPS)), perm
    return Scene(*(np.asarray(getattr(scene, g)).reshape(-1, w)[perm] for g, w in GROUPS)), perm


_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=max(1, min(8, len(os.sched_getaffinity(0)))))
    return _POOL


def upload_f64(a, device) -> torch.Tensor:
    """Host array -> device FP64 tensor through a pinned staging buffer filled
    by several threads (numpy's copy releases the GIL), then one async DMA:
    roughly memory-bandwidth bound instead of the single-threaded pageable
    copy path.  The staging block returns to torch's caching host allocator
    once the copy has completed."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if _registered(a):
        return torch.from_numpy(a).to(device, non_blocking=True)
    h = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    src, dst = a.reshape(-1), h.numpy().reshape(-1)
    n = src.size
    k = 8 if n >= (1 << 20) else 1
    cuts = [n * i // k for i in range(k + 1)]
    if k == 1:
        np.copyto(dst, src)
    else:
        list(_pool().map(lambda i: np.copyto(dst[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]]), range(k)))
    return h.to(device, non_blocking=True)


_SEEN = {}              # (id(owner array), data pointer, bytes) -> [weakref(owner), pointer, bytes, state]
_REGISTER_MIN = 1 << 22  # smaller arrays: the staging copy is cheaper than a registration


def _unregister(ptr):
    from . import _lib
    _lib.lib().sdgr_host_unregister(ptr)


def _registered(a) -> bool:
    """True when `a`'s memory is page-locked for direct DMA.  An array is
    registered (sdgr_host_register) the SECOND time it is uploaded: the
    reference's training loop updates the scene arrays in place
    (optimize.py:206), so they are seen every call, while one-off arrays
    (dL/dS, temporaries) keep the staging path and never pay a registration.
    The registration is dropped when the array is collected.  Arrays whose
    pages overlap another registration fail to register and keep staging."""
    if a.nbytes < _REGISTER_MIN or not a.flags.writeable:
        return False
    owner = a
    while isinstance(owner.base, np.ndarray):   # callers pass fresh reshaped views
        owner = owner.base
    ptr = a.ctypes.data
    key = (id(owner), ptr, a.nbytes)
    ent = _SEEN.get(key)
    if ent is None or ent[0]() is not owner:
        _SEEN[key] = [weakref.ref(owner, lambda _r, k=key: _SEEN.pop(k, None)), ptr, a.nbytes, "seen"]
        return False
    if ent[3] == "seen":
        from . import _lib
        if _lib.lib().sdgr_host_register(ptr, a.nbytes) == 0:
            weakref.finalize(owner, _unregister, ptr).atexit = False
            ent[3] = "pinned"
        else:
            ent[3] = "failed"
    return ent[3] == "pinned"


_STAGE = {}
_POOL_LOCK = threading.Lock()
_OUT_POOL = []                 # [pinned tensor, numpy view of it]: recycled result blocks
_OUT_POOL_BYTES = 1 << 30      # beyond this, results are copied out of one staging block


def _np_dtype(dt):
    return torch.empty(0, dtype=dt).numpy().dtype


def _result_block(total):
    """A page-locked block of >= total bytes that no caller array references
    any more, or None.  Result arrays are numpy views of a block (their .base
    chain ends at the block's array), so the block's reference count is 2
    (pool slot + call argument) exactly when the caller has dropped every
    array -- and every view of them -- handed out from it.  Best fit, so a small image never occupies a gradient block."""
    for attempt in range(2):
        free = [e for e in _OUT_POOL if e[1].nbytes >= total and sys.getrefcount(e[1]) == 2]
        if free:
            best = min(free, key=lambda e: e[1].nbytes)
            if best[1].nbytes <= 4 * total + (1 << 20):   # an image never pins a gradient block
                return best
        if attempt == 0 and any(total <= e[1].nbytes <= 4 * total + (1 << 20) for e in _OUT_POOL):
            # a block of the right size exists but is referenced: results the
            # caller dropped may still be held by a reference cycle of the
            # call's objects (young: generations 0-1).  Collecting them is
            # cheaper than page-locking a new block (~0.4 ms per MB).
            gc.collect(1)
    if sum(e[1].nbytes for e in _OUT_POOL) + total > _OUT_POOL_BYTES:
        return None
    t = torch.empty((max(total, 1 << 20),), dtype=torch.uint8, pin_memory=True)
    _OUT_POOL.append([t, t.numpy()])
    return _OUT_POOL[-1]


def download(tensors) -> list:
    """Device tensors -> numpy arrays the caller owns.  The D2H lands directly
    in a recycled page-locked block and the arrays are views of it (no
    copy-out, no first-touch page faults of fresh memory: the reference's
    training loop drops each call's gradients before the next-but-one call,
    so two blocks cycle).  A block is reused only once nothing references
    it.  Past _OUT_POOL_BYTES of live blocks the arrays are copied out of one
    reused staging block into fresh memory by the thread pool instead."""
    sizes = [t.numel() * t.element_size() for t in tensors]
    total = sum((b + 255) // 256 * 256 for b in sizes)
    with _POOL_LOCK:   # a block is taken (views created) before another caller looks for a free one
        blk = _result_block(total)
        if blk is not None:
            out, o = [], 0
            for t, b in zip(tensors, sizes):
                out.append(blk[1][o:o + b].view(_np_dtype(t.dtype)).reshape(tuple(t.shape)))
                o += (b + 255) // 256 * 256
    if blk is not None:
        o = 0
        for t, b in zip(tensors, sizes):
            blk[0][o:o + b].view(t.dtype).view(t.shape).copy_(t, non_blocking=True)
            o += (b + 255) // 256 * 256
        torch.cuda.current_stream().synchronize()
        return out
    with _POOL_LOCK:
        return _download_staged(tensors, sizes, total)


def _download_staged(tensors, sizes, total) -> list:
    buf = _STAGE.get("d2h")
    if buf is None or buf.numel() < total:
        buf = torch.empty((max(total, 1 << 20),), dtype=torch.uint8, pin_memory=True)
        _STAGE["d2h"] = buf
    views, o = [], 0
    for t, b in zip(tensors, sizes):
        v = buf[o:o + b].view(t.dtype).view(t.shape)
        v.copy_(t, non_blocking=True)
        views.append(v)
        o += (b + 255) // 256 * 256
    torch.cuda.current_stream().synchronize()
    out = [np.empty(tuple(t.shape), dtype=v.numpy().dtype) for t, v in zip(tensors, views)]
    jobs = []
    for src, dst in zip(views, out):
        a, d = src.numpy().reshape(-1), dst.reshape(-1)
        n = a.size
        k = 8 if n >= (1 << 20) else 1
        jobs += [(a, d, n * i // k, n * (i + 1) // k) for i in range(k)]
    list(_pool().map(lambda j: np.copyto(j[1][j[2]:j[3]], j[0][j[2]:j[3]]), jobs))
    return out


def as_device_scene(scene, device=None) -> tuple[DeviceScene, bool]:
    """(device scene, was_host).  Host scenes keep float64 on device so the
    FP64 key chain sees the caller's exact values."""
    if isinstance(scene, DeviceScene):
        return scene, False
    pos = scene.positions
    if isinstance(pos, torch.Tensor) and pos.is_cuda:
        dt = pos.dtype if pos.dtype in (torch.float32, torch.float64) else torch.float64
        return DeviceScene(*(getattr(scene, g).reshape(-1, w).to(dt).contiguous() for g, w in GROUPS)), False
    dev = device or torch.device("cuda", torch.cuda.current_device())
    if isinstance(pos, torch.Tensor):
        return DeviceScene.from_host(scene, dtype=torch.float64, device=dev), True
    return DeviceScene(*(upload_f64(np.reshape(getattr(scene, g), (-1, w)), dev) for g, w in GROUPS)), True
