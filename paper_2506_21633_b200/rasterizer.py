"""SDGR forward + custom backward on B200: the drop-in for sarsplat's hot path.

Public functions keep the reference's names, signatures and error
behaviour (forward.py:138-285, backward.py:86-290):

    render(scene, config, cov_reg=0.3, cutoff=3.0)           -> image
    render_forward(scene, config, cov_reg=0.3, cutoff=3.0)   -> ForwardResult
    backward(fwd, dL_dS)                                     -> SceneGradients
    project_all / build_ray_lists / build_splat_lists /
    compute_intensities / splat_image / grad_image_stage /
    grad_intensity_stage / grad_geometry_stage               (stage functions)

Every stage is a libsdgr call (include/sdgr.h) on the current torch CUDA
stream; torch only provides device memory.  There is no CPU path: without a
GPU or without libsdgr.so these functions raise.

Host scenes (numpy, like the reference's) are uploaded as float64 and the
results come back as numpy float64 arrays, so existing callers work
unchanged.  DeviceScene inputs stay on the device and results are CUDA
tensors (float32).
"""
from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import ptr
from .errors import DeviceError, InvalidParameterError, NumericalError, StateError
from .radar import n_rays, radar_rotation, view_constants
from .scene import GROUPS, DeviceScene, as_device_scene, download, upload_f64

DEFAULT_COV_REG = 0.3
DEFAULT_CUTOFF = 3.0
# Rays stop once their log-transmittance exceeds S_STOP: later pairs would
# contribute < e^-40 * P ~ 4e-18 * P.  float("inf") = the reference's
# exhaustive walk (bit-for-bit the same list traversal).
S_STOP = 40.0
TILE = _lib.TILE
# ~32 depth segments per SM: short segments balance the persistent walks
# (measured on c4: 148*4 -> 567, 148*16 -> 650, 148*32 -> 657, 148*64 -> 635 views/s)
SMS_TARGET_ITEMS = 148 * 32


def _stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check(rc: int, what: str) -> None:
    if rc == _lib.OK:
        return
    msg = _lib.lib().sdgr_status_string(rc).decode()
    if rc == _lib.ERR_INVALID:
        raise InvalidParameterError(f"{what}: {msg}")
    if rc == _lib.ERR_NUMERICAL:
        raise NumericalError(f"{what}: {msg}")
    if rc == _lib.ERR_STATE:
        raise StateError(f"{what}: {msg}")
    raise DeviceError(f"{what}: {msg} (status {rc})")


def _empty(shape, dtype, device):
    return torch.empty(shape, dtype=dtype, device=device)


def _scene_desc(ds: DeviceScene) -> _lib.SceneDesc:
    """POD descriptor of a device scene.  The kernels read raw pointers, so the
    five arrays must share one float dtype and device, be contiguous and have
    shape (n, w) -- anything else is rejected here."""
    arrs = ds.arrays()
    n = len(ds)
    dt, dev = arrs[0].dtype, arrs[0].device
    if dt not in (torch.float32, torch.float64):
        raise InvalidParameterError(f"scene arrays must be float32 or float64, got {dt}")
    for (g, w), a in zip(GROUPS, arrs):
        if a.dtype != dt or a.device != dev:
            raise InvalidParameterError(f"scene.{g}: dtype/device differ from positions ({a.dtype}, {a.device})")
        if tuple(a.shape) != (n, w):
            raise InvalidParameterError(f"scene.{g}: shape {tuple(a.shape)} != ({n}, {w})")
        if not a.is_contiguous():
            raise InvalidParameterError(f"scene.{g}: not contiguous")
    if dev.type != "cuda":
        raise InvalidParameterError("scene arrays must be CUDA tensors")
    d = _lib.SceneDesc()
    d.n = len(ds)
    d.dtype = 0 if ds.dtype == torch.float32 else 1
    d.positions, d.rotations, d.log_scales, d.sh_coeffs, d.ke_raw = (ptr(t) for t in ds.arrays())
    return d


# ----------------------------------------------------------------------------
# projection (K1)
# ----------------------------------------------------------------------------
class _PlaneRecords:
    def __init__(self, n, device, with_cov):
        self.uv = _empty((n, 2), torch.float64, device)
        self.inv_cov = _empty((n, 4), torch.float64, device)
        self.cov = _empty((n, 4), torch.float64, device) if with_cov else None
        self.bbox = _empty((n, 4), torch.int16, device)
        self.cell_mask = _empty((n,), torch.int64, device)
        self.tile_mask = _empty((n,), torch.int64, device)
        self.n_tiles = _empty((n,), torch.int32, device)
        self.packed = None   # gather rows: multi-view steps only
        self.emit = None     # fused count + emit rows: multi-view steps only

    def desc(self) -> _lib.Plane:
        p = _lib.Plane()
        for f, _ in _lib.Plane._fields_:
            setattr(p, f, ptr(getattr(self, f)))
        return p


def _as_out(t, host: bool):
    """Reference-shaped results: numpy for host (numpy) callers, device tensors otherwise."""
    return t.cpu().numpy() if host else t


class Projection:
    """Device projection of one scene into one view (geometry.py:185-230).

    Records are N-sized in scene order; the reference's compacted views
    (``indices``, ``uv_comp``, ...) are exposed as properties that gather the
    visible rows on demand -- numpy arrays when the scene came from the host,
    device tensors otherwise.
    """

    def __init__(self, n: int, device, config, cov_reg: float, cutoff: float, accessors: bool, host: bool = False):
        self.n_scene = n
        self.config = config
        self.cov_reg = cov_reg
        self.cutoff = cutoff
        self.host = host
        self.view = view_constants(config, cov_reg, cutoff)
        self.comp = _PlaneRecords(n, device, accessors)
        self.img = _PlaneRecords(n, device, accessors)
        self.depth_key = _empty((n,), torch.int64, device)
        self.kappa = _empty((n,), torch.float64, device)
        self.phase_f = _empty((n,), torch.float64, device)
        self.phase_raw = _empty((n,), torch.float64, device)
        self.flags = _empty((n,), torch.uint8, device)
        self.counters = torch.zeros((4,), dtype=torch.int32, device=device)
        self.member_pairs = torch.zeros((2,), dtype=torch.int64, device=device)
        self.ke_act = _empty((n, 2), torch.float64, device) if accessors else None
        self.look = _empty((n, 4), torch.float64, device) if accessors else None
        self._vis_idx = None
        self._rows = None
        self._counts = None

    def desc(self) -> _lib.ProjectionDesc:
        d = _lib.ProjectionDesc()
        d.n = self.n_scene
        d.comp = self.comp.desc()
        d.img = self.img.desc()
        d.depth_key, d.kappa, d.phase, d.phase_raw = (
            ptr(self.depth_key), ptr(self.kappa), ptr(self.phase_f), ptr(self.phase_raw))
        d.flags, d.counters, d.ke_act, d.look = ptr(self.flags), ptr(self.counters), ptr(self.ke_act), ptr(self.look)
        d.member_pairs = ptr(self.member_pairs)
        return d

    @classmethod
    def from_planes(cls, config, uv_comp, depth, cov_comp=None, uv_img=None, cov_img=None, ke_sum=None,
                    phase=None, cutoff: float = DEFAULT_CUTOFF, device=None) -> "Projection":
        """A projection given directly in plane space -- the reference tests'
        hand-assembled Projection (tests/test_forward.py:43-59: identity
        covariances, kappa = P = 1 unless given, uv_img = uv_comp) -- with
        the device records built by sdgr_project_planes, so the binning,
        compositing and backward stages run on it unchanged."""
        host = not isinstance(uv_comp, torch.Tensor)
        dev = device or (uv_comp.device if not host else torch.device("cuda", torch.cuda.current_device()))
        f64 = lambda x: (x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))  # noqa: E731
                         ).to(device=dev, dtype=torch.float64).contiguous()
        uv_c = f64(uv_comp).reshape(-1, 2)
        k = uv_c.shape[0]
        if k == 0:
            raise InvalidParameterError("projection is empty")
        eye = torch.eye(2, dtype=torch.float64, device=dev).expand(k, 2, 2)
        cc = f64(cov_comp).reshape(k, 2, 2) if cov_comp is not None else eye
        ci = f64(cov_img).reshape(k, 2, 2) if cov_img is not None else cc
        tri = lambda c: torch.stack([c[:, 0, 0], c[:, 0, 1], c[:, 1, 1]], 1).contiguous()  # noqa: E731
        uv_i = f64(uv_img).reshape(k, 2) if uv_img is not None else uv_c
        kap = f64(ke_sum).reshape(k) if ke_sum is not None else torch.ones(k, dtype=torch.float64, device=dev)
        ph = f64(phase).reshape(k) if phase is not None else torch.ones(k, dtype=torch.float64, device=dev)
        d = f64(depth).reshape(k)
        proj = cls(k, dev, config, 0.0, cutoff, accessors=True, host=host)
        proj._desc = proj.desc()
        keep = (uv_c, uv_i, d, tri(cc), tri(ci), ph, kap)
        _check(_lib.lib().sdgr_project_planes(C.byref(proj.view), k, *(ptr(t) for t in keep), C.byref(proj._desc),
                                              _stream()), "sdgr_project_planes")
        proj._keep = keep
        proj.ke_act[:, 0] = kap / 2.0
        proj.ke_act[:, 1] = kap / 2.0
        proj.look[:] = torch.tensor([0.0, 0.0, 1.0, 1.0], dtype=torch.float64, device=dev)
        return proj

    # -- reference-shaped accessors (compacted to the K visible rows) -------
    @property
    def visible(self) -> torch.Tensor:
        return (self.flags & _lib.FLAG_VISIBLE) != 0

    @property
    def idx_t(self) -> torch.Tensor:
        """Visible scene indices (device tensor), ascending."""
        if self._vis_idx is None:
            self._vis_idx = torch.nonzero(self.visible).flatten()
        return self._vis_idx

    @property
    def row_of(self) -> torch.Tensor:
        """Scene index -> projection row (device; -1 for invisible rows)."""
        if self._rows is None:
            v = self.visible.to(torch.int64)
            self._rows = torch.where(self.visible, torch.cumsum(v, 0) - 1, torch.full_like(v, -1))
        return self._rows

    @property
    def indices(self):
        return _as_out(self.idx_t, self.host)

    def __len__(self) -> int:
        return int(self.idx_t.numel())

    def _counts_host(self):
        if self._counts is None:
            self._counts = self.counters.cpu().tolist()
        return self._counts

    @property
    def n_culled(self) -> int:
        return int(self._counts_host()[2])

    @property
    def n_skipped(self) -> int:
        return int(self._counts_host()[1])

    def _k(self, t):
        return _as_out(t[self.idx_t], self.host)

    @property
    def uv_comp(self):
        return self._k(self.comp.uv)

    @property
    def uv_img(self):
        return self._k(self.img.uv)

    @property
    def depth(self):
        return _as_out(decode_depth(self.depth_key[self.idx_t]), self.host)

    def _cov(self, pl):
        if pl.cov is None:
            raise StateError("projection was built without covariance accessors")
        c = pl.cov[self.idx_t]
        return _as_out(torch.stack([torch.stack([c[:, 0], c[:, 1]], -1), torch.stack([c[:, 1], c[:, 2]], -1)], -2),
                       self.host)

    @property
    def cov_comp(self):
        return self._cov(self.comp)

    @property
    def cov_img(self):
        return self._cov(self.img)

    @property
    def phase(self):
        return self._k(self.phase_f)

    @property
    def phase_unclamped(self):
        return self._k(self.phase_raw)

    @property
    def ke_sum(self):
        return self._k(self.kappa)

    @property
    def ke_fwd(self):
        return self._k(self.ke_act[:, 0])

    @property
    def ke_bwd(self):
        return self._k(self.ke_act[:, 1])

    @property
    def look_dirs(self):
        return self._k(self.look[:, :3])

    @property
    def look_dists(self):
        return self._k(self.look[:, 3])

    @property
    def rotation(self) -> np.ndarray:
        return radar_rotation(self.config.azimuth_deg, self.config.elevation_deg)


def decode_depth(key: torch.Tensor) -> torch.Tensor:
    """Inverse of the device depth key (common.cuh:depth_key)."""
    k = key.clone()
    neg = k >= 0  # sign bit clear in the key <=> negative depth
    k = torch.where(neg, ~k, k ^ torch.tensor(-0x8000000000000000, dtype=torch.int64, device=k.device))
    return k.view(torch.float64)


def project_all(scene, config, cov_reg: float = DEFAULT_COV_REG, cutoff: float = DEFAULT_CUTOFF,
                accessors: bool = True) -> Projection:
    """geometry.project_all (geometry.py:233-340) on the device."""
    if len(scene) == 0:
        raise InvalidParameterError("scene is empty")
    ds, host = as_device_scene(scene)
    return _project(ds, config, cov_reg, cutoff, accessors, host)


def _project(ds: DeviceScene, config, cov_reg, cutoff, accessors, host: bool = False) -> Projection:
    proj = Projection(len(ds), ds.device, config, cov_reg, cutoff, accessors, host=host)
    proj._desc = proj.desc()
    sd = _scene_desc(ds)
    _check(_lib.lib().sdgr_project(C.byref(sd), C.byref(proj.view), C.byref(proj._desc), _stream()),
           "sdgr_project")
    return proj


# ----------------------------------------------------------------------------
# binning (K2-K5)
# ----------------------------------------------------------------------------
@dataclass
class TileLists:
    """Per-16x16-tile key lists of one plane, plus the reference's per-cell
    pair view of the same plane.

    Device key lists (what the kernels walk): `pair_tile` / `tile_prim` /
    `tile_range` -- per tile, the scene indices with a member cell in the
    tile, in (depth, index) order on the computation plane (plane 0) and
    index order on the imaging plane (plane 1).

    Reference view (forward.RayLists / SplatPairs, forward.py:112-135,
    202-210), materialised on first access by sdgr_cell_pairs: `pair_cell`
    (`pair_pixel`), `pair_prim` (projection rows), `delta`, `q`, `weight`,
    `offsets`, `cell_list(iu, iv)` and len() = member pairs.

    Buffers hold `capacity` tile pairs.  With a cached capacity
    (device_count) the exact count stays on the device (`count_dev`) until
    n_pairs is read.
    """

    plane: int
    n_u: int
    n_v: int
    tiles_x: int
    tiles_y: int
    capacity: int
    pair_tile: torch.Tensor
    pair_pos: torch.Tensor
    tile_prim: torch.Tensor
    pre_prim: torch.Tensor
    pair_start: torch.Tensor
    tile_range: torch.Tensor
    seg_len: int
    max_items: int
    items: torch.Tensor
    tile_first: torch.Tensor
    n_items: torch.Tensor
    pair_rec: torch.Tensor | None = None
    member_pairs: int | None = None   # member (cell, Gaussian) pairs of the plane (capacity bound)
    count_dev: torch.Tensor | None = None   # device_count mode: offsets[n] on the device
    projection: "Projection | None" = None
    _n_host: int | None = None
    _desc: object = field(default=None, repr=False)
    _cells: dict | None = field(default=None, repr=False)

    @property
    def n_pairs(self) -> int:
        """(tile, Gaussian) pairs of the plane."""
        if self._n_host is None:
            self._n_host = int(self.count_dev.item())
        return self._n_host

    @property
    def n_tiles(self) -> int:
        return self.tiles_x * self.tiles_y

    def desc(self) -> _lib.TilesDesc:
        if self._desc is None:
            d = _lib.TilesDesc()
            d.plane, d.tiles_x, d.tiles_y, d.n_tiles = self.plane, self.tiles_x, self.tiles_y, self.n_tiles
            d.n_pairs = self.capacity
            d.device_count = 0 if self.count_dev is None else 1
            d.pair_tile, d.pair_pos, d.pair_prim = ptr(self.pair_tile), ptr(self.pair_pos), ptr(self.tile_prim)
            d.pre_prim, d.pair_start, d.tile_range = ptr(self.pre_prim), ptr(self.pair_start), ptr(self.tile_range)
            d.seg_len, d.max_items = self.seg_len, self.max_items
            d.items, d.tile_first, d.n_items = ptr(self.items), ptr(self.tile_first), ptr(self.n_items)
            d.pair_rec = ptr(self.pair_rec)
            self._desc = d
        return self._desc

    def tile_list(self, tx: int, ty: int) -> torch.Tensor:
        t = ty * self.tiles_x + tx
        s, e = self.tile_range[t].tolist()
        return self.tile_prim[s:e]

    # -- reference view: member (cell, Gaussian) pairs ---------------------
    def cells(self) -> dict:
        """Device arrays of the member pairs in the reference's order:
        cell, prim (scene index), row (projection row), delta, q, w, offsets."""
        if self._cells is None:
            p = self.projection
            if p is None:
                raise StateError("tile lists without their projection")
            lib, st, dev = _lib.lib(), _stream(), self.tile_range.device
            n_cells = self.n_u * self.n_v
            off = torch.zeros((n_cells + 1,), dtype=torch.int64, device=dev)
            desc = self.desc()
            _check(lib.sdgr_cell_pairs(C.byref(p._desc), C.byref(p.view), C.byref(desc), ptr(off), None, None, None,
                                       None, st), "sdgr_cell_pairs")
            t = int(off[-1].item())
            prim = _empty((max(t, 1),), torch.int32, dev)
            delta = _empty((max(t, 1), 2), torch.float64, dev)
            q = _empty((max(t, 1),), torch.float64, dev)
            w = _empty((max(t, 1),), torch.float64, dev)
            if t:
                _check(lib.sdgr_cell_pairs(C.byref(p._desc), C.byref(p.view), C.byref(desc), ptr(off), ptr(prim),
                                           ptr(delta), ptr(q), ptr(w), st), "sdgr_cell_pairs")
            cell = torch.repeat_interleave(torch.arange(n_cells, device=dev), off[1:] - off[:-1])
            prim, delta, q, w = prim[:t], delta[:t], q[:t], w[:t]
            self._cells = dict(cell=cell, prim=prim, row=p.row_of[prim.long()], delta=delta, q=q, w=w, offsets=off)
        return self._cells

    def _ref(self, key):
        host = self.projection.host if self.projection is not None else False
        return _as_out(self.cells()[key], host)

    @property
    def pair_cell(self):
        return self._ref("cell")

    @property
    def pair_pixel(self):
        return self._ref("cell")

    @property
    def pair_prim(self):
        """Projection rows of the member pairs (RayLists.pair_prim)."""
        return self._ref("row")

    @property
    def delta(self):
        return self._ref("delta")

    @property
    def q(self):
        return self._ref("q")

    @property
    def weight(self):
        return self._ref("w")

    @property
    def offsets(self):
        return self._ref("offsets")

    def cell_list(self, iu: int, iv: int):
        """Projection rows covering cell (iu, iv), shallow-to-deep (RayLists.cell_list)."""
        c = self.cells()
        a, b = c["offsets"][iv * self.n_u + iu: iv * self.n_u + iu + 2].tolist()
        return _as_out(c["row"][a:b], self.projection.host)

    def __len__(self) -> int:
        return int(self.cells()["cell"].numel())


def _seg_len(n_pairs: int) -> int:
    if os.environ.get("SDGR_SEG_LEN"):          # A/B override (profiling)
        return int(min(max(int(os.environ["SDGR_SEG_LEN"]), 256), 8192)) // 256 * 256
    seg = -(-n_pairs // SMS_TARGET_ITEMS)
    seg = -(-seg // 256) * 256
    return int(min(max(seg, 256), 8192))


# Pair capacities per (N, ray grid, image, cutoff, plane) from the last exact
# binning: later calls of the same shape allocate from them and keep the pair
# counts on the device (no host round trip inside render_forward).  A call
# whose counts outgrow them is detected on the device and re-binned exactly.
_CAPS: dict = {}
CAP_HEADROOM = 1.25


class _Binner:
    """Runs K2-K5 for the requested planes."""

    def __init__(self, proj: Projection):
        self.proj = proj
        self.lib = _lib.lib()
        self.dev = proj.flags.device

    def _key(self, pl):
        v = self.proj.view
        return (self.proj.n_scene, v.n_u, v.n_v, v.n_az, v.n_rg, float(v.cutoff), pl)

    def _lists(self, pl, cap, count_dev=None):
        p, dev, n = self.proj, self.dev, self.proj.n_scene
        v = p.view
        nu, nv = (v.n_u, v.n_v) if pl == 0 else (v.n_az, v.n_rg)
        tx, ty = -(-nu // TILE), -(-nv // TILE)
        seg = _seg_len(cap)
        max_items = -(-cap // seg) + tx * ty
        c = max(int(cap), 1)
        return TileLists(
            plane=pl, n_u=nu, n_v=nv, tiles_x=tx, tiles_y=ty, capacity=int(cap),
            pair_tile=_empty((c,), torch.int32, dev), pair_pos=_empty((c,), torch.int32, dev),
            tile_prim=_empty((c,), torch.int32, dev), pre_prim=_empty((c,), torch.int32, dev),
            pair_start=_empty((n,), torch.int32, dev), tile_range=_empty((tx * ty, 2), torch.int32, dev),
            seg_len=seg, max_items=max_items, items=_empty((max_items, 4), torch.int32, dev),
            tile_first=_empty((tx * ty,), torch.int32, dev),
            n_items=torch.zeros((4,), dtype=torch.int32, device=dev),
            pair_rec=(_empty((c, _lib.PAIR_REC_BYTES), torch.uint8, dev) if pl == 0 else None),
            count_dev=count_dev, projection=p, _n_host=None if count_dev is not None else int(cap))

    def run(self, planes=(0, 1), exact: bool = False):
        if not exact and all(self._key(pl) in _CAPS for pl in planes):
            return self._run_cached(planes)
        return self._run_exact(planes)

    def _depth_order(self, ws, ws_bytes, st):
        order = _empty((self.proj.n_scene,), torch.int32, self.dev)
        _check(self.lib.sdgr_depth_order(C.byref(self.proj._desc), ptr(order), ptr(ws), ws_bytes, st),
               "sdgr_depth_order")
        return order

    def _run_exact(self, planes):
        """Counts first, one host read of the totals, then exactly sized lists."""
        p, lib, st, dev = self.proj, self.lib, _stream(), self.dev
        n = p.n_scene
        ws_bytes = lib.sdgr_workspace_bytes(n, 1)
        ws = _empty((ws_bytes,), torch.uint8, dev)
        order = self._depth_order(ws, ws_bytes, st) if 0 in planes else None
        offsets = {}
        for pl in planes:
            off = _empty((n + 1,), torch.int32, dev)
            _check(lib.sdgr_count_pairs(C.byref(p._desc), pl, ptr(order) if pl == 0 else None, ptr(off),
                                        ptr(ws), ws_bytes, st), "sdgr_count_pairs")
            offsets[pl] = off
        host = torch.cat([torch.stack([offsets[pl][n] for pl in planes]).to(torch.int64), p.member_pairs]).cpu()
        totals = host[: len(planes)].tolist()
        member = host[len(planes):].tolist()
        ws_bytes = lib.sdgr_workspace_bytes(n, max(max(totals), 1))
        ws = _empty((ws_bytes,), torch.uint8, dev)
        out = {}
        for pl, total in zip(planes, totals):
            tl = self._lists(pl, int(total))
            _check(lib.sdgr_bin_pairs(C.byref(p._desc), C.byref(p.view), ptr(order) if pl == 0 else None,
                                      ptr(offsets[pl]), C.byref(tl.desc()), ptr(ws), ws_bytes, st),
                   "sdgr_bin_pairs")
            tl.member_pairs = int(member[pl])
            _CAPS[self._key(pl)] = (int(total * CAP_HEADROOM) + 1024, int(member[pl] * CAP_HEADROOM) + 1024)
            out[pl] = tl
        self.order = order
        return out

    def _run_cached(self, planes):
        """Cached capacities: depth order + fused count/emit/sort per plane
        (sdgr_bin_batch of one view), counts left on the device."""
        p, lib, st, dev = self.proj, self.lib, _stream(), self.dev
        n = p.n_scene
        caps = {pl: _CAPS[self._key(pl)] for pl in planes}
        ws_bytes = lib.sdgr_batch_workspace_bytes(n, max(c for c, _ in caps.values()), 1)
        ws = _empty((ws_bytes,), torch.uint8, dev)
        order = self._depth_order(ws, ws_bytes, st) if 0 in planes else None
        out = {}
        for pl in planes:
            off = _empty((n + 1,), torch.int32, dev)
            tl = self._lists(pl, caps[pl][0], count_dev=off[n])
            tl.member_pairs = caps[pl][1]
            tls = (_lib.TilesDesc * 1)(tl.desc())
            orders = (C.c_void_p * 1)(ptr(order) if pl == 0 else None)
            offs = (C.c_void_p * 1)(ptr(off))
            _check(lib.sdgr_bin_batch(1, C.byref(p._desc), C.byref(p.view), pl, orders if pl == 0 else None,
                                      offs, tls, ptr(ws), ws_bytes, st), "sdgr_bin_batch")
            out[pl] = tl
        self.order = order
        return out


def build_ray_lists(projection: Projection, config=None) -> TileLists:
    """Computation-plane tile lists (forward.build_ray_lists, forward.py:138-155)."""
    return _Binner(projection).run((0,))[0]


def build_splat_lists(projection: Projection, config=None) -> TileLists:
    """Imaging-plane tile lists (forward._build_splat_pairs, forward.py:213-224)."""
    return _Binner(projection).run((1,))[1]


# ----------------------------------------------------------------------------
# forward compositing (K6, K7)
# ----------------------------------------------------------------------------
@dataclass
class IntensityBuffer:
    """Per-Gaussian intensities (N-sized, scene order) + per-ray segment state.

    Reference view (forward.IntensityBuffer, forward.py:167-175): `intensity`
    (K rows) and the per-member-pair `tau`, `trans`, `absorb`, `contrib` in
    the RayLists pair order, computed on first access (sdgr_cell_intensities)."""

    intensity_n: torch.Tensor
    seg_sum: torch.Tensor
    seg_base: torch.Tensor
    partial: torch.Tensor
    status: torch.Tensor
    s_stop: float
    projection: "Projection | None" = None   # set when the reference's compacted views are wanted
    replay: "ReplayLog | None" = None
    replay_ok: bool | None = None            # host copy of "the log did not overflow" (one status read)
    rays: "TileLists | None" = None
    _pairs: dict | None = None

    @property
    def indices(self):
        return None if self.projection is None else self.projection.indices

    @property
    def intensity(self):
        """(K,) compacted like the reference's IntensityBuffer.intensity."""
        if self.projection is None:
            return self.intensity_n
        return _as_out(self.intensity_n[self.projection.idx_t], self.projection.host)

    def _pair(self, key):
        if self._pairs is None:
            if self.rays is None or self.projection is None:
                raise StateError("per-pair buffers need the ray lists and the projection")
            c = self.rays.cells()
            t = c["prim"].numel()
            dev = self.intensity_n.device
            out = {k: _empty((max(t, 1),), torch.float64, dev) for k in ("tau", "trans", "absorb", "contrib")}
            p = self.projection
            _check(_lib.lib().sdgr_cell_intensities(C.byref(p._desc), self.rays.n_u * self.rays.n_v,
                                                    ptr(c["offsets"]), ptr(c["prim"]), ptr(c["w"]),
                                                    ptr(out["tau"]), ptr(out["trans"]), ptr(out["absorb"]),
                                                    ptr(out["contrib"]), _stream()), "sdgr_cell_intensities")
            self._pairs = {k: v[:t] for k, v in out.items()}
        return _as_out(self._pairs[key], self.projection.host)

    @property
    def tau(self):
        return self._pair("tau")

    @property
    def trans(self):
        return self._pair("trans")

    @property
    def absorb(self):
        return self._pair("absorb")

    @property
    def contrib(self):
        return self._pair("contrib")


class ReplayLog:
    """Buffers of the live-pair log (sdgr_replay, include/sdgr.h): written by
    the forward walk, replayed by the backward so it touches live pairs only."""

    def __init__(self, capacity: int, max_items: int, seg_len: int, device, n_pairs: int = 1):
        cap = int(max(capacity, 1))
        self.capacity = cap
        self.desc_per_item = 40 * max(1, -(-seg_len // 256))
        self.y1 = _empty((cap,), torch.float64, device)
        self.t2 = _empty((cap,), torch.float64, device)
        self.w = _empty((cap,), torch.float64, device)
        self.j = _empty((cap,), torch.uint8, device)
        self.r = _empty((cap,), torch.uint8, device)
        self.desc = _empty((max(max_items, 1) * self.desc_per_item, 4), torch.int32, device)
        self.desc_count = torch.zeros((max(max_items, 1),), dtype=torch.int32, device=device)
        self.cursor = torch.zeros((2,), dtype=torch.int64, device=device)
        self.gpair = _empty((max(int(n_pairs), 1),), torch.float64, device)
        d = _lib.ReplayDesc()
        d.capacity, d.desc_per_item = cap, self.desc_per_item
        d.y1, d.t2, d.w, d.j, d.r = ptr(self.y1), ptr(self.t2), ptr(self.w), ptr(self.j), ptr(self.r)
        d.desc, d.desc_count, d.cursor = ptr(self.desc), ptr(self.desc_count), ptr(self.cursor)
        d.gpair = ptr(self.gpair)
        self.desc_c = d

    def overflowed(self) -> bool:
        return bool(self.cursor[1].item())


def compute_intensities(rays: TileLists, projection: Projection, s_stop: float = S_STOP,
                        check: bool = True, replay: bool = True) -> IntensityBuffer:
    """forward.compute_intensities (forward.py:178-199) on the device.
    check=True reads the status once and raises NumericalError like the
    reference (forward.py:192-196)."""
    dev = projection.flags.device
    n = projection.n_scene
    cap = max(rays.max_items, 1) * 256
    buf = IntensityBuffer(
        intensity_n=_empty((n,), torch.float64, dev),
        seg_sum=_empty((cap,), torch.float64, dev),
        seg_base=_empty((cap,), torch.float64, dev),
        partial=_empty((max(rays.capacity, 1),), torch.float64, dev),
        status=torch.zeros((4,), dtype=torch.int32, device=dev),
        s_stop=float(s_stop),
        projection=projection, rays=rays,
    )
    if replay and rays.member_pairs is not None:
        buf.replay = ReplayLog(rays.member_pairs, rays.max_items, rays.seg_len, dev, rays.capacity)
    _check(_lib.lib().sdgr_composite_forward(
        C.byref(projection.view), C.byref(projection._desc), C.byref(rays.desc()), float(s_stop),
        ptr(buf.seg_sum), ptr(buf.seg_base), ptr(buf.partial), ptr(buf.intensity_n), ptr(buf.status),
        C.byref(buf.replay.desc_c) if buf.replay else None, _stream()),
        "sdgr_composite_forward")
    if check:
        ov, bad = _forward_status(buf, projection, [rays])
        if ov:
            raise OverflowError("pair capacity exceeded")
        if bad:
            raise NumericalError(f"non-finite intensity at primitive {_first_bad_primitive(projection)}")
    return buf


def _forward_status(buf: IntensityBuffer, proj: Projection, lists) -> tuple[bool, bool]:
    """ONE host read per forward: (binning overflow, non-finite intensity);
    also records whether the replay log overflowed.  A Gaussian with a
    non-finite phase or extinction poisons every member pair it has in the
    reference, even behind an opaque ray (forward.py:188-196), so besides
    the walk's own flag a visible Gaussian with non-finite P or kappa counts
    when it has a member cell (checked on the error path only)."""
    words = [buf.status[0].to(torch.int64), (~torch.isfinite(buf.intensity_n)).any().to(torch.int64)]
    if proj.phase_f is not None and proj.kappa is not None:
        words.append((proj.visible & ~(torch.isfinite(proj.phase_f) & torch.isfinite(proj.kappa))).any()
                     .to(torch.int64))
    else:
        words.append(torch.zeros((), dtype=torch.int64, device=buf.status.device))
    words += [tl.n_items[1].to(torch.int64) for tl in lists]
    if buf.replay is not None:
        words.append(buf.replay.cursor[1])
    f = torch.stack(words).cpu().tolist()
    if buf.replay is not None:
        buf.replay_ok = not f.pop()
    ov = any(f[3:])
    bad = bool(f[0] or f[1]) or (bool(f[2]) and _first_bad_primitive(proj) >= 0)
    return ov, bad


def _first_bad_primitive(proj: Projection) -> int:
    """The primitive the reference names (forward.py:193-196): the first
    non-finite pair in (cell, depth, index) order.  Every member pair of a
    Gaussian with non-finite P or kappa is non-finite, so it is the bad
    Gaussian minimising (first member cell, depth, index).  Error path only."""
    bad = proj.visible & ~(torch.isfinite(proj.phase_f) & torch.isfinite(proj.kappa))
    cand = torch.nonzero(bad).flatten().cpu().numpy()
    if cand.size == 0:
        return -1
    v = proj.view
    uv = proj.comp.uv.cpu().numpy()
    A = proj.comp.inv_cov.cpu().numpy()
    bb = proj.comp.bbox.cpu().numpy().astype(np.int64)
    dk = proj.depth_key.cpu().numpy().view(np.uint64)
    cut2 = v.cutoff * v.cutoff
    best = None
    for g in cand:
        x0, x1, y0, y1 = bb[g]
        first = None
        for iv in range(y0, y1 + 1):
            for iu in range(x0, x1 + 1):
                dx, dy = iu - uv[g, 0], iv - uv[g, 1]
                q = A[g, 0] * dx * dx + 2.0 * A[g, 1] * dx * dy + A[g, 2] * dy * dy
                if not math.isfinite(v.cutoff) or q <= cut2:
                    first = iv * v.n_u + iu
                    break
            if first is not None:
                break
        if first is None:
            continue
        key = (first, int(dk[g]), int(g))
        if best is None or key < best:
            best = key
    return -1 if best is None else best[2]


def splat_image(intensities: IntensityBuffer, projection: Projection, config=None,
                pairs: TileLists | None = None):
    """forward.splat_image (forward.py:227-240): (n_range, n_azimuth) float64
    (numpy for host callers).

    Gaussian-parallel with deterministic fixed-point accumulation; the
    imaging-plane tile lists (``pairs``) are not needed and are ignored."""
    return _as_out(_splat(intensities, projection), projection.host)


def _splat(intensities: IntensityBuffer, projection: Projection) -> torch.Tensor:
    v = projection.view
    dev = projection.flags.device
    image = _empty((v.n_rg, v.n_az), torch.float64, dev)
    scratch = _empty((v.n_rg * v.n_az + 1,), torch.int64, dev)
    _check(_lib.lib().sdgr_splat(C.byref(v), C.byref(projection._desc), ptr(intensities.intensity_n),
                                 ptr(scratch), ptr(image), _stream()), "sdgr_splat")
    return image


class ForwardResult:
    """A rendered image plus every buffer the backward pass needs (forward.py:243-253).

    The imaging-plane tile lists (`splat`) are built on first access: the
    splat and its backward are Gaussian-parallel and never read them."""

    def __init__(self, scene, device_scene, config, projection, rays, intensities, image_t, host=False,
                 splat=None):
        self.scene, self.device_scene, self.config = scene, device_scene, config
        self.projection, self.rays, self.intensities = projection, rays, intensities
        self.image_t, self.host = image_t, host
        self._splat = splat
        self._image_host = None

    @property
    def splat(self) -> TileLists:
        if self._splat is None:
            self._splat = _Binner(self.projection).run((1,), exact=True)[1]
        return self._splat

    @property
    def image(self):
        if not self.host:
            return self.image_t
        if self._image_host is None:
            self._image_host = download([self.image_t])[0]
        return self._image_host


def render_forward(scene, config, cov_reg: float = DEFAULT_COV_REG, cutoff: float = DEFAULT_CUTOFF,
                   s_stop: float = S_STOP, accessors: bool = True) -> ForwardResult:
    """Render and retain the buffers for backward (forward.py:256-273).

    One host round trip per call (the status word: non-finite intensity,
    capacity overflow); pair buffers are sized from the capacities of the
    last call of the same shape.  Host scenes get the image as numpy FP64."""
    if len(scene) == 0:
        raise NumericalError("cannot retain buffers for an empty scene")
    ds, host = as_device_scene(scene)
    proj = _project(ds, config, cov_reg, cutoff, accessors, host)
    for exact in (False, True):
        rays = _Binner(proj).run((0,), exact=exact)[0]
        buf = compute_intensities(rays, proj, s_stop=s_stop, check=False)
        image = _splat(buf, proj)
        ov, bad = _forward_status(buf, proj, [rays])
        if not ov:
            break
        _CAPS.pop(_Binner(proj)._key(0), None)   # grown footprints: re-bin with exact counts
    if bad:
        raise NumericalError(f"non-finite intensity at primitive {_first_bad_primitive(proj)}")
    if not accessors:
        buf.projection = None
    return ForwardResult(scene=scene, device_scene=ds, config=config, projection=proj, rays=rays,
                         intensities=buf, image_t=image, host=host)


def render(scene, config, cov_reg: float = DEFAULT_COV_REG, cutoff: float = DEFAULT_CUTOFF,
           s_stop: float = S_STOP):
    """Forward-render into an (n_range, n_azimuth) image (forward.py:276-285)."""
    host = not (isinstance(scene, DeviceScene) or (isinstance(scene.positions, torch.Tensor)
                                                   and scene.positions.is_cuda))
    if len(scene) == 0:
        img = torch.zeros((config.n_range, config.n_azimuth), dtype=torch.float64)
        return img.double().numpy() if host else img.cuda()
    return render_forward(scene, config, cov_reg, cutoff, s_stop=s_stop, accessors=False).image


# ----------------------------------------------------------------------------
# backward (K8-K10)
# ----------------------------------------------------------------------------
@dataclass
class SceneGradients:
    """Per-primitive gradients + densification statistic (backward.py:25-50)."""

    positions: object
    rotations: object
    log_scales: object
    sh_coeffs: object
    ke_raw: object
    uv_grad_norm: object
    visible: object

    def param_arrays(self):
        return (self.positions, self.rotations, self.log_scales, self.sh_coeffs, self.ke_raw)

    @classmethod
    def zeros_device(cls, n: int, device, dtype=torch.float32) -> "SceneGradients":
        z = lambda *s: torch.zeros(s, dtype=dtype, device=device)  # noqa: E731
        return cls(z(n, 3), z(n, 4), z(n, 3), z(n, 16), z(n, 2), z(n),
                   torch.zeros((n,), dtype=torch.int32, device=device))

    def desc(self) -> _lib.GradsDesc:
        arrays = self.param_arrays() + (self.uv_grad_norm,)
        dt = arrays[0].dtype
        if dt not in (torch.float32, torch.float64) or any(a.dtype != dt or not a.is_contiguous() for a in arrays):
            raise InvalidParameterError("gradient arrays must be contiguous and share float32 or float64")
        if self.visible.dtype not in (torch.int32, dt):
            raise InvalidParameterError("visible counts must be int32 or the gradient dtype")
        d = _lib.GradsDesc()
        d.dtype = 0 if dt == torch.float32 else 1
        d.visible_dtype = 0 if self.visible.dtype == torch.int32 else 1
        d.positions, d.rotations, d.log_scales = ptr(self.positions), ptr(self.rotations), ptr(self.log_scales)
        d.sh_coeffs, d.ke_raw = ptr(self.sh_coeffs), ptr(self.ke_raw)
        d.uv_grad_norm, d.visible = ptr(self.uv_grad_norm), ptr(self.visible)
        return d

    def to_numpy(self) -> "SceneGradients":
        """FP64 numpy copies (the reference's SceneGradients layout), through
        one reused pinned staging buffer (scene.download)."""
        arrays = [a.double() for a in self.param_arrays()] + [self.uv_grad_norm.double(), self.visible > 0]
        return SceneGradients(*download(arrays))


# -- fused device stages (what backward() runs) ------------------------------
def image_stage_sums(fwd: ForwardResult, dL_dS: torch.Tensor) -> torch.Tensor:
    """grad_image_stage's per-Gaussian sums, acc (6, N) float64 = [dL/dI,
    G00, G01, G11, dL/du, dL/dv] on the imaging plane (G: the quadratic-form
    gradient before the inverse chain)."""
    p = fwd.projection
    acc = _empty((6, p.n_scene), torch.float64, p.flags.device)
    _check(_lib.lib().sdgr_grad_image(C.byref(p.view), C.byref(p._desc), ptr(fwd.intensities.intensity_n),
                                      ptr(dL_dS), ptr(acc), _stream()), "sdgr_grad_image")
    return acc


def intensity_stage_partials(fwd: ForwardResult, dL_dI: torch.Tensor, use_replay: bool = True) -> torch.Tensor:
    """grad_intensity_stage's per-(tile, Gaussian) partials (T16, 8) float64
    = [dL/dP, dL/dkappa, G00, G01, G11, dL/du, dL/dv, 0] on the computation
    plane, indexed by pre-sort position.  dL_dI: (N,) scene order."""
    p, rays, buf = fwd.projection, fwd.rays, fwd.intensities
    dev = p.flags.device
    partial = _empty((max(rays.capacity, 1), 8), torch.float64, dev)
    cap = max(rays.max_items, 1) * 256
    seg_g = _empty((cap,), torch.float64, dev)
    seg_d = _empty((cap,), torch.float64, dev)
    ok = buf.replay_ok if buf.replay_ok is not None else (buf.replay is not None and not buf.replay.overflowed())
    rp = buf.replay if (use_replay and buf.replay is not None and ok) else None
    _check(_lib.lib().sdgr_grad_intensity(C.byref(p.view), C.byref(p._desc), C.byref(rays.desc()),
                                          buf.s_stop, ptr(buf.seg_base), ptr(dL_dI), ptr(seg_g), ptr(seg_d),
                                          ptr(partial), C.byref(rp.desc_c) if rp else None, _stream()),
           "sdgr_grad_intensity")
    return partial


def geometry_stage_fused(fwd: ForwardResult, acc_img: torch.Tensor, partial_comp: torch.Tensor,
                         out: SceneGradients | None = None, accumulate: bool = False) -> SceneGradients:
    """grad_geometry_stage + grad_sh_stage + final scatter (backward.py:171-290)
    from the fused stage sums.  Host (FP64) callers get FP64 gradients like
    the reference; device callers float32 unless they pass `out`."""
    p = fwd.projection
    if out is None:
        out = SceneGradients.zeros_device(p.n_scene, p.flags.device,
                                          dtype=torch.float64 if fwd.host else torch.float32)
    sd = _scene_desc(fwd.device_scene)
    gd = out.desc()
    _check(_lib.lib().sdgr_grad_geometry(C.byref(sd), C.byref(p.view), C.byref(p._desc),
                                         C.byref(fwd.rays.desc()), ptr(acc_img), ptr(partial_comp),
                                         C.byref(gd), int(accumulate), _stream()), "sdgr_grad_geometry")
    return out


# -- reference-shaped stage functions (backward.py:86-240) ------------------
def _stage_grads(fwd: ForwardResult, plane: int, src: torch.Tensor) -> torch.Tensor:
    p = fwd.projection
    out = _empty((8, p.n_scene), torch.float64, p.flags.device)
    _check(_lib.lib().sdgr_stage_grads(C.byref(p._desc), plane, C.byref(fwd.rays.desc()) if plane == 0 else None,
                                       ptr(src), ptr(out), _stream()), "sdgr_stage_grads")
    return out


def _to_n(fwd: ForwardResult, x, width: int | None = None) -> torch.Tensor:
    """K-row (reference layout) input -> N-row device FP64 in scene order."""
    p = fwd.projection
    dev = p.flags.device
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    t = t.to(device=dev, dtype=torch.float64)
    shape = (p.n_scene,) + tuple(t.shape[1:])
    out = torch.zeros(shape, dtype=torch.float64, device=dev)
    out[p.idx_t] = t
    return out


def grad_image_stage(fwd: ForwardResult, dL_dS):
    """backward.grad_image_stage (backward.py:86-104): the reference's
    4-tuple (dL/dI (K,), dL/dbeta (T_i,) per imaging pair in SplatPairs
    order, dL/dcov_img (K, 2, 2), dL/duv_img (K, 2))."""
    g = _as_device_grad(dL_dS, fwd)
    acc = image_stage_sums(fwd, g)
    st = _stage_grads(fwd, 1, acc)
    sp = fwd.splat.cells()
    t = sp["prim"].numel()
    dbeta = _empty((max(t, 1),), torch.float64, g.device)
    _check(_lib.lib().sdgr_splat_pair_grads(t, ptr(sp["cell"].to(torch.int32)), ptr(sp["prim"]), ptr(g),
                                            ptr(fwd.intensities.intensity_n), ptr(dbeta), _stream()),
           "sdgr_splat_pair_grads")
    idx, host = fwd.projection.idx_t, fwd.projection.host
    return tuple(_as_out(a, host) for a in (st[0][idx], dbeta[:t], st[2:6][:, idx].T.reshape(-1, 2, 2),
                                            st[6:8][:, idx].T))


def grad_intensity_stage(fwd: ForwardResult, dL_dI):
    """backward.grad_intensity_stage (backward.py:107-148): the reference's
    4-tuple (dL/dP (K,), dL/dke_sum (K,), dL/dcov_comp (K, 2, 2),
    dL/duv_comp (K, 2)) for a K-row dL/dI."""
    partial = intensity_stage_partials(fwd, _to_n(fwd, dL_dI))
    st = _stage_grads(fwd, 0, partial)
    idx, host = fwd.projection.idx_t, fwd.projection.host
    return tuple(_as_out(a, host) for a in (st[0][idx], st[1][idx], st[2:6][:, idx].T.reshape(-1, 2, 2),
                                            st[6:8][:, idx].T))


def _explicit_geometry(fwd: ForwardResult, dcov_c=None, dcov_i=None, duv_c=None, duv_i=None, dP=None,
                       dke=None) -> SceneGradients:
    p = fwd.projection
    if fwd.device_scene is None:
        raise StateError("the geometry stage needs the scene the projection came from")
    n, dev = p.n_scene, p.flags.device
    ex = torch.zeros((14, n), dtype=torch.float64, device=dev)
    if dcov_c is not None:
        ex[0:4] = _to_n(fwd, np.asarray(dcov_c).reshape(-1, 4) if not isinstance(dcov_c, torch.Tensor)
                        else dcov_c.reshape(-1, 4)).T
    if dcov_i is not None:
        ex[4:8] = _to_n(fwd, np.asarray(dcov_i).reshape(-1, 4) if not isinstance(dcov_i, torch.Tensor)
                        else dcov_i.reshape(-1, 4)).T
    if duv_c is not None:
        ex[8:10] = _to_n(fwd, duv_c).T
    if duv_i is not None:
        ex[10:12] = _to_n(fwd, duv_i).T
    if dP is not None:
        ex[12] = _to_n(fwd, dP)
    if dke is not None:
        ex[13] = _to_n(fwd, dke)
    out = SceneGradients.zeros_device(n, dev, dtype=torch.float64)
    _check(_lib.lib().sdgr_grad_geometry_explicit(C.byref(_scene_desc(fwd.device_scene)), C.byref(p.view),
                                                  C.byref(p._desc), ptr(ex.contiguous()), C.byref(out.desc()),
                                                  _stream()), "sdgr_grad_geometry_explicit")
    return out


def grad_geometry_stage(fwd: ForwardResult, dL_dcov_comp, dL_dcov_img, dL_duv_comp, dL_duv_img, dL_dP):
    """backward.grad_geometry_stage (backward.py:171-232): plane-space
    gradients (K rows) -> (dL/dpos (K, 3), dL/drot (K, 4), dL/dlogs (K, 3))."""
    g = _explicit_geometry(fwd, dL_dcov_comp, dL_dcov_img, dL_duv_comp, dL_duv_img, dL_dP)
    idx = fwd.projection.idx_t
    host = fwd.projection.host
    return tuple(_as_out(a[idx], host) for a in (g.positions, g.rotations, g.log_scales))


def grad_sh_stage(fwd: ForwardResult, dL_dP):
    """backward.grad_sh_stage (backward.py:235-240): (K, 16) SH-coefficient
    gradients, zero where the phase clamp is active."""
    g = _explicit_geometry(fwd, dP=dL_dP)
    return _as_out(g.sh_coeffs[fwd.projection.idx_t], fwd.projection.host)


def _as_device_grad(dL_dS, fwd: ForwardResult) -> torch.Tensor:
    dev = fwd.projection.flags.device
    if isinstance(dL_dS, torch.Tensor):
        return dL_dS.to(device=dev, dtype=torch.float64).contiguous()
    return upload_f64(dL_dS, dev)


def backward(fwd: ForwardResult, dL_dS, out: SceneGradients | None = None, accumulate: bool = False,
             validate: bool = True, use_replay: bool = True) -> SceneGradients:
    """Full backward from an image gradient (backward.py:243-290).

    use_replay=False re-walks the tile lists instead of replaying the forward's
    live-pair log (both are parity-tested; the replay is the fast path)."""
    shape = tuple(dL_dS.shape)
    img_shape = (fwd.projection.view.n_rg, fwd.projection.view.n_az)
    if shape != img_shape:
        raise StateError(f"image gradient shape {shape} does not match forward {img_shape}")
    if fwd.scene is None or fwd.projection.n_scene != len(fwd.scene):
        raise StateError("scene changed since the forward pass; buffers are stale")
    if validate:
        # host arrays are checked on the host (no device round trip)
        ok = (bool(np.all(np.isfinite(dL_dS))) if not isinstance(dL_dS, torch.Tensor)
              else bool(torch.isfinite(dL_dS).all().item()))
        if not ok:
            raise InvalidParameterError("dL_dS contains non-finite values")
    g = _as_device_grad(dL_dS, fwd)
    acc_img = image_stage_sums(fwd, g)
    partial = intensity_stage_partials(fwd, acc_img[0], use_replay=use_replay)
    grads = geometry_stage_fused(fwd, acc_img, partial, out=out, accumulate=accumulate)
    return grads.to_numpy() if fwd.host and out is None else grads


def forward_from_projection(projection: Projection, s_stop: float = S_STOP, scene=None) -> ForwardResult:
    """A ForwardResult for a given projection (tests/test_backward.py:18-27
    builds one from a synthetic Projection): binning, compositing and the
    splat on the device; the geometry stages need `scene`."""
    rays = _Binner(projection).run((0,), exact=True)[0]
    buf = compute_intensities(rays, projection, s_stop=s_stop)
    image = _splat(buf, projection)
    ds = None if scene is None else as_device_scene(scene)[0]
    return ForwardResult(scene=scene, device_scene=ds, config=projection.config, projection=projection, rays=rays,
                         intensities=buf, image_t=image, host=projection.host)


def launch_count() -> int:
    """Kernels libsdgr has launched in this process."""
    return int(_lib.lib().sdgr_launch_count())
