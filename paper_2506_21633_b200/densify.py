"""Densification on the device: GradAccumulator and
densify_and_prune of the reference's training loop.

Reference: `optimize.GradAccumulator` (optimize.py:217-239),
`optimize.densify_and_prune` (optimize.py:251-312),
`optimize.AdamState.reindex` (optimize.py:162-168).  The per-Gaussian
decisions, clone displacement, split sampling (x += chol(Sigma) xi) and prune
test run as kernels (csrc/densify.cu); the row gathers use the index lists
the flags define; xi is drawn from the caller's numpy generator exactly as
the reference draws it, so a seeded run reproduces the reference's children.
Densification changes N, so it runs between (not inside) captured steps.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ptr
from .rasterizer import SceneGradients, _check, _scene_desc, _stream
from .scene import GROUPS, DeviceScene


@dataclass
class DensifyConfig:
    """The TrainConfig fields densify_and_prune reads (optimize.py:30-70 defaults)."""

    densify_grad_threshold: float = 3e-3
    max_radius_factor: float = 0.3
    clone_size_factor: float = 0.01
    prune_phase_floor: float = 5e-3
    split_scale_shrink: float = 1.6


@dataclass
class DensifyEvent:
    iteration: int
    n_cloned: int
    n_split: int
    n_pruned: int
    n_after: int


class GradAccumulator:
    """Densification statistics between densify events (optimize.py:217-239), FP64 on the device."""

    def __init__(self, norm_sum: torch.Tensor, pos_sum: torch.Tensor, count: torch.Tensor):
        self.norm_sum, self.pos_sum, self.count = norm_sum, pos_sum, count

    @classmethod
    def zeros(cls, n: int, device="cuda") -> "GradAccumulator":
        z = lambda *s: torch.zeros(s, dtype=torch.float64, device=device)  # noqa: E731
        return cls(z(n), z(n, 3), z(n))

    def update(self, grads: SceneGradients) -> None:
        """grads: device SceneGradients (visible = views that saw each Gaussian)."""
        gd = grads.desc()
        _check(_lib.lib().sdgr_accum_update(C.byref(gd), int(self.count.shape[0]), ptr(self.norm_sum),
                                            ptr(self.pos_sum), ptr(self.count), _stream()), "sdgr_accum_update")

    def mean_norm(self) -> torch.Tensor:
        return self.norm_sum / torch.clamp(self.count, min=1.0)

    def mean_pos_grad(self) -> torch.Tensor:
        return self.pos_sum / torch.clamp(self.count, min=1.0)[:, None]


def _gather(scene: DeviceScene, idx: torch.Tensor) -> DeviceScene:
    return DeviceScene(*(a.index_select(0, idx) for a in scene.arrays()))


def _concat(parts) -> DeviceScene:
    return DeviceScene(*(torch.cat([getattr(p, g) for p in parts]) for g, _ in GROUPS))


def densify_and_prune(scene: DeviceScene, accum: GradAccumulator, config, view, scene_extent: float,
                      position_lr: float, rng: np.random.Generator, state=None):
    """optimize.densify_and_prune on a DeviceScene.  Returns (new scene,
    fresh accumulator, DensifyEvent); `state` (train.AdamState) is reindexed
    in place like AdamState.reindex: originals keep their moments, clones and
    children start at zero, then the survivors are selected."""
    lib, st, dev = _lib.lib(), _stream(), scene.device
    n = len(scene)
    cap = config.max_radius_factor * view.ground_extent_m
    flags = torch.empty((n,), dtype=torch.uint8, device=dev)
    sd = _scene_desc(scene)
    _check(lib.sdgr_densify_flags(C.byref(sd), ptr(accum.norm_sum), ptr(accum.count), float(cap),
                                  float(config.clone_size_factor * scene_extent),
                                  float(config.densify_grad_threshold), ptr(flags), st), "sdgr_densify_flags")
    kept_idx = torch.nonzero(flags != 2).flatten()
    clone_idx = torch.nonzero(flags == 1).flatten()
    split_idx = torch.nonzero(flags == 2).flatten()
    parts = [_gather(scene, kept_idx)]
    n_clone, n_split = int(clone_idx.numel()), int(split_idx.numel())
    if n_clone:
        clones = _gather(scene, clone_idx)
        pos_sum = accum.pos_sum.index_select(0, clone_idx).contiguous()
        count = accum.count.index_select(0, clone_idx).contiguous()
        cd = _scene_desc(clones)
        _check(lib.sdgr_clone_shift(C.byref(cd), ptr(pos_sum), ptr(count), float(position_lr), st),
               "sdgr_clone_shift")
        parts.append(clones)
    if n_split:
        children = _gather(scene, split_idx.repeat_interleave(2))
        xi = torch.from_numpy(rng.normal(size=(len(children), 3))).to(dev)   # the reference's draw
        chd = _scene_desc(children)
        _check(lib.sdgr_split_children(C.byref(chd), ptr(xi), float(math.log(config.split_scale_shrink)), st),
               "sdgr_split_children")
        parts.append(children)
    merged = _concat(parts) if len(parts) > 1 else parts[0]
    survive = torch.empty((len(merged),), dtype=torch.uint8, device=dev)
    md = _scene_desc(merged)
    _check(lib.sdgr_prune_flags(C.byref(md), float(cap), float(config.prune_phase_floor), ptr(survive), st),
           "sdgr_prune_flags")
    keep = torch.nonzero(survive).flatten()
    result = _gather(merged, keep)
    n_pruned = len(merged) - int(keep.numel())
    if state is not None:
        n_new = n_clone + 2 * n_split
        for mom in (state.m, state.v):
            for g, _ in GROUPS:
                a = getattr(mom, g)
                kept_rows = a.index_select(0, kept_idx)
                pad = torch.zeros((n_new,) + tuple(a.shape[1:]), dtype=a.dtype, device=dev)
                setattr(mom, g, torch.cat([kept_rows, pad]).index_select(0, keep))
    event = DensifyEvent(iteration=-1, n_cloned=n_clone, n_split=n_split, n_pruned=n_pruned, n_after=len(result))
    return result, GradAccumulator.zeros(len(result), dev), event
