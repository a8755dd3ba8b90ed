"""Device versions of the steps either side of the path in the reference's
training loop: the loss with its SSIM gradient and the
Adam update, so render -> loss -> backward -> update runs without a host
round trip (and inside a CUDA graph).

Reference: `optimize.loss` (optimize.py:85-102), `metrics.ssim_with_grad`
(metrics.py:98-137), `optimize.AdamState` / `adam_step` (optimize.py:141-207).
Compute is in the C ABI (`sdgr_loss`, `sdgr_adam_step`, csrc/train.cu); this
module mirrors the reference's Python signatures.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import ptr
from .errors import InvalidParameterError
from .rasterizer import SceneGradients, _check, _scene_desc, _stream
from .scene import DeviceScene

SSIM_WIN_SIZE = 11
SSIM_SIGMA = 1.5
PARAM_GROUPS = ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")


def ssim_kernel() -> np.ndarray:
    """The normalised 11-tap Gaussian (metrics._ssim_kernel, metrics.py:45-49)."""
    r = (SSIM_WIN_SIZE - 1) // 2
    t = np.arange(-r, r + 1, dtype=np.float64)
    k = np.exp(-(t * t) / (2.0 * SSIM_SIGMA * SSIM_SIGMA))
    return k / k.sum()


class LossBuffers:
    """Device scratch of `loss` for one image shape (reusable across calls)."""

    def __init__(self, h: int, w: int, device="cuda"):
        self.h, self.w = int(h), int(w)
        lib = _lib.lib()
        self.scratch = torch.empty((lib.sdgr_loss_scratch_bytes(self.h, self.w),), dtype=torch.uint8, device=device)
        self.kernel = (C.c_double * SSIM_WIN_SIZE)(*ssim_kernel())  # host taps (baked into the launch)
        self.value = torch.zeros((), dtype=torch.float64, device=device)

    def run(self, rendered: torch.Tensor, target: torch.Tensor, grad: torch.Tensor, lambda_ssim: float,
            max_val: float) -> None:
        _check(_lib.lib().sdgr_loss(ptr(rendered), ptr(target), self.h, self.w, float(lambda_ssim), float(max_val),
                                    C.cast(self.kernel, C.c_void_p), ptr(self.value), ptr(grad),
                                    ptr(self.scratch), _stream()),
               "sdgr_loss")


def loss(rendered, target, lambda_ssim: float = 0.2, max_val: float = 1.0, buffers: LossBuffers | None = None):
    """optimize.loss (optimize.py:85-102): ((1-l) L1 + l (1-SSIM), dL/dS).

    numpy inputs -> (float, numpy float64) like the reference; CUDA tensors ->
    (0-d device tensor, device tensor), no host synchronisation."""
    host = not isinstance(rendered, torch.Tensor)
    S = torch.as_tensor(np.asarray(rendered, dtype=np.float64) if host else rendered, dtype=torch.float64)
    Y = torch.as_tensor(np.asarray(target, dtype=np.float64) if not isinstance(target, torch.Tensor) else target,
                        dtype=torch.float64)
    if S.shape != Y.shape or S.dim() != 2:
        raise InvalidParameterError(f"shape mismatch: {tuple(S.shape)} vs {tuple(Y.shape)}")
    if not (0.0 <= lambda_ssim <= 1.0):
        raise InvalidParameterError("lambda_ssim must lie in [0, 1]")
    dev = S.device if S.is_cuda else torch.device("cuda")
    S, Y = S.to(dev).contiguous(), Y.to(dev).contiguous()
    buf = buffers if buffers is not None else LossBuffers(*S.shape, device=dev)
    grad = torch.empty_like(S)
    buf.run(S, Y, grad, lambda_ssim, max_val)
    if host:
        return float(buf.value.item()), grad.cpu().numpy()
    return buf.value.clone(), grad


@dataclass
class AdamState:
    """First/second moments per parameter group (optimize.AdamState,
    optimize.py:141-168), device tensors shaped like the scene's."""

    m: DeviceScene
    v: DeviceScene
    step: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    skipped: torch.Tensor = field(default=None)  # device u64 count of zeroed non-finite entries

    @classmethod
    def for_scene(cls, scene: DeviceScene) -> "AdamState":
        z = lambda: DeviceScene(*(torch.zeros_like(a) for a in scene.arrays()))  # noqa: E731
        return cls(m=z(), v=z(), skipped=torch.zeros((), dtype=torch.int64, device=scene.device))

    @property
    def n_skipped(self) -> int:
        return int(self.skipped.item())


def adam_step(scene: DeviceScene, grads: SceneGradients, state: AdamState, lrs: dict,
              displacement_bound: float | None = None, guard: torch.Tensor | None = None) -> None:
    """optimize.adam_step (optimize.py:171-207), in place on the device scene.

    grads: device SceneGradients (float32, e.g. MultiViewStep.grads).  The
    bias corrections use the host step count (as the reference does).
    guard: optional device int32 scalar; the kernel skips the whole update
    when it is non-zero (MultiViewStep.overflow)."""
    state.step += 1
    b1, b2 = state.beta1, state.beta2
    bc1 = 1.0 - b1 ** state.step
    bc2 = 1.0 - b2 ** state.step
    lr = (C.c_double * 5)(*(float(lrs[g]) for g in PARAM_GROUPS))
    sd, md, vd = _scene_desc(scene), _scene_desc(state.m), _scene_desc(state.v)
    gd = grads.desc()
    bound = float(displacement_bound) if displacement_bound is not None else -1.0
    _check(_lib.lib().sdgr_adam_step(C.byref(sd), C.byref(gd), C.byref(md), C.byref(vd), lr, float(b1), float(b2),
                                     float(state.eps), bc1, bc2, bound, ptr(state.skipped),
                                     ptr(guard) if guard is not None else None, _stream()),
           "sdgr_adam_step")


class TrainStep:
    """One optimiser step over a set of views, entirely on the device: for
    every view render -> loss vs its target -> backward (MultiViewStep with
    targets), the gradient sum (all-reduced across ranks when distributed),
    the SH-degree mask, and Adam -- the multi-view form of the body of
    optimize.train (optimize.py:395-425; one view per step there).  The view
    work is one CUDA graph per step; Adam is one more kernel."""

    def __init__(self, scene: DeviceScene, configs, targets: torch.Tensor, lambda_ssim: float = 0.2,
                 max_val: float = 1.0, **kw):
        from .multiview import MultiViewStep
        self.scene = scene
        self.mv = MultiViewStep(scene, configs, targets=targets, lambda_ssim=lambda_ssim, max_val=max_val, **kw)
        self.dlds = torch.zeros(targets.shape, dtype=torch.float64, device=scene.device)
        self.state = AdamState.for_scene(scene)
        self.graph_generation = -1

    def __call__(self, lrs: dict, sh_active: int = 16, displacement_bound: float | None = None,
                 use_graph: bool = True, check: bool = True) -> torch.Tensor:
        """Returns the per-view loss values (device tensor, before the update).

        The Adam kernel is guarded on the device by the step's overflow word,
        so a step whose pair buffers overflowed (footprints grew past the
        calibrated capacity) never moves the parameters.  With check=True
        (one host read per step) such a step is recalibrated -- which also
        drops the stale graph -- and re-run on the unchanged scene, so the
        update applied is exactly the one a large enough buffer gives."""
        for attempt in range(3):
            self._step(lrs, sh_active, displacement_bound, use_graph)
            if not check:
                break
            bad, ov = torch.stack([self.mv.status[0], self.mv.overflow]).cpu().tolist()
            if not ov:
                if bad:
                    from .errors import NumericalError
                    raise NumericalError("non-finite intensity in a training step")
                break
            self.state.step -= 1          # the guarded update did not happen
            self.mv.calibrate()           # larger buffers; drops the captured graph
        else:
            raise OverflowError("pair capacity still exceeded after recalibration")
        return self.mv.loss_values

    def _step(self, lrs, sh_active, displacement_bound, use_graph):
        if use_graph:
            if self.mv.graph is None or self.graph_generation != self.mv.generation:
                self.mv.capture(self.dlds)
                self.graph_generation = self.mv.generation
            self.mv.graph_step()
        else:
            self.mv.run(self.dlds, check=False)
        g = self.mv.grads
        if sh_active < 16:
            g.sh_coeffs[:, sh_active:] = 0.0   # optimize.py:412-413
        adam_step(self.scene, g, self.state, lrs, displacement_bound, guard=self.mv.overflow)
