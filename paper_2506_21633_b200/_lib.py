"""ctypes binding of libsdgr.so (the C ABI declared in include/sdgr.h).

This module is the only place the shared library is loaded.  There is no
fallback: if the library is missing or its ABI version does not match,
importing the rasterizer raises ImportError.  Build it with
``python -m paper_2506_21633_b200.csrc.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

ABI_VERSION = 2
import os  # noqa: E402

# SDGR_LIB selects a profiling build (e.g. libsdgr_prof.so) of the same ABI
LIB_PATH = Path(__file__).resolve().parent / os.environ.get("SDGR_LIB", "libsdgr.so")

OK, ERR_INVALID, ERR_NUMERICAL, ERR_STATE, ERR_CUDA, ERR_CAPACITY = range(6)
FLAG_VISIBLE, FLAG_SKIPPED, FLAG_CULLED = 1, 2, 4
TILE = 16
MAX_BATCH = 24  # default build's SDGR_MAX_BATCH; lib().sdgr_max_batch() is authoritative
PROFILE_KERNELS = 16
K_PROJECT, K_ONESWEEP, K_EMIT, K_GATHER, K_SEGSUM, K_WALK, K_SPLAT, K_GRAD_IMAGE, K_REPLAY_GSUM, K_REPLAY_GRAD, \
    K_GEOMETRY = range(1, 12)
KERNEL_NAMES = {K_PROJECT: "k_project", K_ONESWEEP: "k_onesweep", K_EMIT: "k_count_emit", K_GATHER: "k_gather_prim",
                K_SEGSUM: "k_segsum", K_WALK: "k_walk<kContrib>", K_SPLAT: "k_splat", K_GRAD_IMAGE: "k_grad_image",
                K_REPLAY_GSUM: "k_replay<kGSum>", K_REPLAY_GRAD: "k_replay<kGrad>", K_GEOMETRY: "k_grad_geometry"}

_p = C.c_void_p


class View(C.Structure):
    _fields_ = [
        ("R", C.c_double * 9), ("T", C.c_double * 3), ("cam", C.c_double * 3),
        ("mc", C.c_double * 6), ("mi", C.c_double * 6),
        ("den_u", C.c_double), ("den_v", C.c_double), ("off_vi", C.c_double),
        ("cov_reg", C.c_double), ("cutoff", C.c_double),
        ("n_u", C.c_int32), ("n_v", C.c_int32), ("n_az", C.c_int32), ("n_rg", C.c_int32),
    ]


class SceneDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("dtype", C.c_int32), ("pad_", C.c_int32),
        ("positions", _p), ("rotations", _p), ("log_scales", _p), ("sh_coeffs", _p), ("ke_raw", _p),
    ]


class Plane(C.Structure):
    _fields_ = [
        ("uv", _p), ("inv_cov", _p), ("cov", _p), ("bbox", _p),
        ("cell_mask", _p), ("tile_mask", _p), ("n_tiles", _p), ("packed", _p), ("emit", _p),
    ]


class ProjectionDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("comp", Plane), ("img", Plane),
        ("depth_key", _p), ("kappa", _p), ("phase", _p), ("phase_raw", _p),
        ("flags", _p), ("counters", _p), ("ke_act", _p), ("look", _p), ("member_pairs", _p),
    ]


class ReplayDesc(C.Structure):
    _fields_ = [
        ("capacity", C.c_int64), ("y1", _p), ("t2", _p), ("w", _p), ("j", _p), ("r", _p),
        ("desc_per_item", C.c_int32), ("pad_", C.c_int32), ("desc", _p), ("desc_count", _p), ("cursor", _p),
        ("gpair", _p),
    ]


class TilesDesc(C.Structure):
    _fields_ = [
        ("plane", C.c_int32), ("tiles_x", C.c_int32), ("tiles_y", C.c_int32), ("n_tiles", C.c_int32),
        ("n_pairs", C.c_int64), ("pair_tile", _p), ("pair_pos", _p), ("pair_prim", _p),
        ("pre_prim", _p), ("pair_start", _p), ("tile_range", _p),
        ("seg_len", C.c_int32), ("max_items", C.c_int32), ("device_count", C.c_int32), ("pad_", C.c_int32),
        ("items", _p), ("tile_first", _p),
        ("n_items", _p), ("pair_rec", _p),
    ]


PAIR_REC_BYTES = 80  # sizeof(sdgr_pair_rec)


class GradsDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("visible_dtype", C.c_int32),
        ("positions", _p), ("rotations", _p), ("log_scales", _p), ("sh_coeffs", _p),
        ("ke_raw", _p), ("uv_grad_norm", _p), ("visible", _p),
    ]


# (name, restype, argtypes) for every symbol include/sdgr.h declares
SIGNATURES = [
    ("sdgr_version", C.c_int, []),
    ("sdgr_status_string", C.c_char_p, [C.c_int]),
    ("sdgr_launch_count", C.c_uint64, []),
    ("sdgr_max_batch", C.c_int, []),
    ("sdgr_workspace_bytes", C.c_size_t, [C.c_int64, C.c_int64]),
    ("sdgr_profile_begin", C.c_int, [C.c_uint32]),
    ("sdgr_profile_end", C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    ("sdgr_profile_timeline", C.c_int, [C.c_int, _p, _p, _p]),
    ("sdgr_host_register", C.c_int, [_p, C.c_size_t]),
    ("sdgr_exp_check", C.c_int, [C.c_int64, _p, _p, _p]),
    ("sdgr_host_unregister", C.c_int, [_p]),
    ("sdgr_project", C.c_int, [C.POINTER(SceneDesc), C.POINTER(View), C.POINTER(ProjectionDesc), _p]),
    ("sdgr_depth_order", C.c_int, [C.POINTER(ProjectionDesc), _p, _p, C.c_size_t, _p]),
    ("sdgr_count_pairs", C.c_int, [C.POINTER(ProjectionDesc), C.c_int32, _p, _p, _p, C.c_size_t, _p]),
    ("sdgr_bin_pairs", C.c_int, [C.POINTER(ProjectionDesc), C.POINTER(View), _p, _p,
                                 C.POINTER(TilesDesc), _p, C.c_size_t, _p]),
    ("sdgr_batch_workspace_bytes", C.c_size_t, [C.c_int64, C.c_int64, C.c_int]),
    ("sdgr_project_batch", C.c_int, [C.POINTER(SceneDesc), C.c_int, C.POINTER(View), C.POINTER(ProjectionDesc),
                                     _p]),
    ("sdgr_depth_order_batch", C.c_int, [C.c_int, C.POINTER(ProjectionDesc), C.POINTER(_p), _p, C.c_size_t,
                                         _p]),
    ("sdgr_bin_batch", C.c_int, [C.c_int, C.POINTER(ProjectionDesc), C.POINTER(View), C.c_int32,
                                 C.POINTER(_p), C.POINTER(_p), C.POINTER(TilesDesc), _p, C.c_size_t, _p]),
    ("sdgr_composite_forward", C.c_int, [C.POINTER(View), C.POINTER(ProjectionDesc), C.POINTER(TilesDesc),
                                         C.c_double, _p, _p, _p, _p, _p, C.POINTER(ReplayDesc), _p]),
    ("sdgr_splat", C.c_int, [C.POINTER(View), C.POINTER(ProjectionDesc), _p, _p, _p, _p]),
    ("sdgr_grad_image", C.c_int, [C.POINTER(View), C.POINTER(ProjectionDesc), _p, _p, _p, _p]),
    ("sdgr_grad_intensity", C.c_int, [C.POINTER(View), C.POINTER(ProjectionDesc), C.POINTER(TilesDesc),
                                      C.c_double, _p, _p, _p, _p, _p, C.POINTER(ReplayDesc), _p]),
    ("sdgr_grad_geometry", C.c_int, [C.POINTER(SceneDesc), C.POINTER(View), C.POINTER(ProjectionDesc),
                                     C.POINTER(TilesDesc), _p, _p, C.POINTER(GradsDesc), C.c_int, _p]),
    ("sdgr_grad_geometry_batch", C.c_int, [C.POINTER(SceneDesc), C.c_int, C.POINTER(View),
                                           C.POINTER(ProjectionDesc), C.POINTER(TilesDesc), C.POINTER(_p),
                                           C.POINTER(_p), C.POINTER(GradsDesc), C.c_int, _p]),
    ("sdgr_grid_workspace_bytes", C.c_size_t, [C.c_int64, C.c_int64]),
    ("sdgr_nn_sqdist", C.c_int, [_p, C.c_int64, _p, C.c_int64, C.POINTER(C.c_double), C.c_double,
                                 C.POINTER(C.c_int32), _p, _p, C.c_size_t, _p]),
    ("sdgr_dbscan", C.c_int, [_p, C.c_int64, C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_int32),
                              C.c_double, C.c_int32, _p, _p, C.c_size_t, _p]),
    ("sdgr_ply_pack", C.c_int, [C.POINTER(SceneDesc), _p, _p]),
    ("sdgr_ply_unpack", C.c_int, [_p, C.c_int64, C.c_int, C.POINTER(C.c_int32), C.POINTER(SceneDesc), _p]),
    ("sdgr_accum_update", C.c_int, [C.POINTER(GradsDesc), C.c_int64, _p, _p, _p, _p]),
    ("sdgr_densify_flags", C.c_int, [C.POINTER(SceneDesc), _p, _p, C.c_double, C.c_double, C.c_double, _p, _p]),
    ("sdgr_clone_shift", C.c_int, [C.POINTER(SceneDesc), _p, _p, C.c_double, _p]),
    ("sdgr_split_children", C.c_int, [C.POINTER(SceneDesc), _p, C.c_double, _p]),
    ("sdgr_prune_flags", C.c_int, [C.POINTER(SceneDesc), C.c_double, C.c_double, _p, _p]),
    ("sdgr_loss_scratch_bytes", C.c_size_t, [C.c_int, C.c_int]),
    ("sdgr_loss", C.c_int, [_p, _p, C.c_int, C.c_int, C.c_double, C.c_double, _p, _p, _p, _p, _p]),
    ("sdgr_cell_pairs", C.c_int, [C.POINTER(ProjectionDesc), C.POINTER(View), C.POINTER(TilesDesc), _p, _p, _p,
                                  _p, _p, _p]),
    ("sdgr_cell_intensities", C.c_int, [C.POINTER(ProjectionDesc), C.c_int64, _p, _p, _p, _p, _p, _p, _p, _p]),
    ("sdgr_splat_pair_grads", C.c_int, [C.c_int64, _p, _p, _p, _p, _p, _p]),
    ("sdgr_stage_grads", C.c_int, [C.POINTER(ProjectionDesc), C.c_int32, C.POINTER(TilesDesc), _p, _p, _p]),
    ("sdgr_grad_geometry_explicit", C.c_int, [C.POINTER(SceneDesc), C.POINTER(View), C.POINTER(ProjectionDesc),
                                              _p, C.POINTER(GradsDesc), _p]),
    ("sdgr_project_planes", C.c_int, [C.POINTER(View), C.c_int64, _p, _p, _p, _p, _p, _p, _p,
                                      C.POINTER(ProjectionDesc), _p]),
    ("sdgr_adam_step", C.c_int, [C.POINTER(SceneDesc), C.POINTER(GradsDesc), C.POINTER(SceneDesc),
                                 C.POINTER(SceneDesc), C.POINTER(C.c_double), C.c_double, C.c_double,
                                 C.c_double, C.c_double, C.c_double, C.c_double, _p, _p, _p]),
]


def load(path: Path | str = LIB_PATH) -> C.CDLL:
    path = Path(path)
    if not path.exists():
        raise ImportError(
            f"libsdgr.so not found at {path}; build it with "
            "`python -m paper_2506_21633_b200.csrc.build` (there is no CPU fallback)")
    lib = C.CDLL(str(path))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sdgr_version() != ABI_VERSION:
        raise ImportError(f"libsdgr ABI {lib.sdgr_version()} != expected {ABI_VERSION}")
    return lib


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None for None)."""
    return None if t is None else t.data_ptr()
