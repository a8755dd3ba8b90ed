"""B200-native SAR Differentiable Gaussian Rasterizer (SDGR).

Drop-in for the hot path of the reference package ``sarsplat``
(render / render_forward / backward and their stage functions), computed by
hand-written sm_100a CUDA kernels behind the C ABI in include/sdgr.h.

    import paper_2506_21633_b200 as sdgr
    fwd = sdgr.render_forward(scene, config)          # scene: sarsplat-style Scene
    grads = sdgr.backward(fwd, dL_dS)                 # SceneGradients

The rasterizer modules load libsdgr.so lazily on first use and raise if it
is missing -- there is no CPU fallback.
"""
from .errors import (DegenerateProjectionError, DeviceError, DivergenceError, InvalidParameterError,
                     NumericalError, SarsplatError, StateError)
from .radar import RadarConfig, radar_position, radar_rotation, view_constants
from .scene import DeviceScene, Scene, spatial_order, spatial_sort

__version__ = "0.1.0"

_LAZY = {
    "render", "render_forward", "backward", "project_all", "build_ray_lists", "build_splat_lists",
    "compute_intensities", "splat_image", "grad_image_stage", "grad_intensity_stage",
    "grad_geometry_stage", "grad_sh_stage", "forward_from_projection", "ForwardResult", "SceneGradients",
    "Projection", "TileLists", "image_stage_sums", "intensity_stage_partials", "geometry_stage_fused",
    "IntensityBuffer", "launch_count", "S_STOP", "DEFAULT_COV_REG", "DEFAULT_CUTOFF",
}


def __getattr__(name):
    if name in _LAZY:
        from . import rasterizer
        return getattr(rasterizer, name)
    if name in ("MultiViewStep", "shard_views"):
        from . import multiview
        return getattr(multiview, name)
    raise AttributeError(name)


__all__ = sorted(_LAZY | {"RadarConfig", "Scene", "DeviceScene", "radar_position", "radar_rotation",
                          "view_constants", "SarsplatError", "InvalidParameterError",
                          "DegenerateProjectionError", "NumericalError", "StateError",
                          "DivergenceError", "DeviceError", "MultiViewStep", "shard_views",
                          "spatial_order", "spatial_sort"})
