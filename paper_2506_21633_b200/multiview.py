"""Multi-view SDGR steps: forward + backward over many views, one all-reduce.

This is the reconstruction-loop shape of the reference's caller
(optimize.train, optimize.py:395-425) scaled out: every rank holds the full
(replicated) Gaussian scene, renders and back-propagates its own shard of the
SAR views with gradients accumulated on the device, and the per-Gaussian
gradients are summed across ranks with one NCCL all-reduce per step
(SURVEY.md §8e).  GradAccumulator semantics (optimize.py:229-233) are kept by
summing uv_grad_norm and visible counts too.

Per view the whole chain -- K1 preprocess, K2-K5 binning, K6/K7 forward,
K8-K10 backward -- is launched with no host round trip: pair buffers use
capacities cached from a calibration pass and the exact counts stay on the
device.  Capacity overflow is detected on the device and folded into one
overflow word per step (`MultiViewStep.overflow`): check() raises
OverflowError from it, and TrainStep recalibrates and re-runs the step (its
Adam update is guarded by the same word on the device, so an overflowed step
never moves the parameters).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import ptr
from .errors import NumericalError, StateError
from .radar import view_constants
from .rasterizer import (DEFAULT_COV_REG, DEFAULT_CUTOFF, S_STOP, ReplayLog, SceneGradients, TILE, _check, _empty,
                         _scene_desc, _seg_len, _stream)
from .scene import DeviceScene

MULTIVIEW_SEG_LEN = 2048  # depth-segment floor for concurrent multi-view steps
GRAD_WIDTH = 30  # 3 + 4 + 3 + 16 + 2 + uv_grad_norm + visible count (float32, exact below 2^24)


def shard_views(configs, rank: int, world: int):
    """Views for `rank`: {v : v mod world == rank} (interleaves elevations)."""
    return [c for i, c in enumerate(configs) if i % world == rank]


GRAD_GROUPS = (3, 4, 3, 16, 2, 1)  # positions, rotations, log_scales, sh_coeffs, ke_raw, uv_grad_norm


def grad_views(flat: torch.Tensor, n: int) -> SceneGradients:
    """SceneGradients whose fields are SoA views into one (30 n,) float32
    buffer; the last n words hold the visible counts as float32 (integers
    below 2^24 are exact, so summing them in float32 is exact)."""
    parts, o = [], 0
    for w in GRAD_GROUPS:
        parts.append(flat[o:o + w * n].view(n, w) if w > 1 else flat[o:o + n])
        o += w * n
    return SceneGradients(*parts, flat[o:o + n])


def allreduce_grads(flat: torch.Tensor, n: int, group=None) -> None:
    """One-step gradient exchange: ONE all-reduce (sum) of the flat float32
    buffer -- every gradient group, uv_grad_norm and the visible counts --
    over all ranks (NCCL on GPU, gloo on CPU): 120 B per Gaussian."""
    import torch.distributed as dist
    dist.all_reduce(flat[: GRAD_WIDTH * n], group=group)


@dataclass
class _PlaneBufs:
    offsets: torch.Tensor
    tiles: object  # TilesDesc
    t: dict


class MultiViewStep:
    """Forward + backward of a list of views with on-device accumulation."""

    def __init__(self, scene: DeviceScene, configs, cov_reg: float = DEFAULT_COV_REG,
                 cutoff: float = DEFAULT_CUTOFF, s_stop: float = S_STOP, headroom: float = 1.3,
                 group=None, geo_batch: int | None = None, lanes: int = 8, targets: torch.Tensor | None = None,
                 ramp: int | None = None,
                 lambda_ssim: float = 0.2, max_val: float = 1.0):
        self.scene = scene
        self.configs = list(configs)
        self.views = [view_constants(c, cov_reg, cutoff) for c in self.configs]
        self.s_stop = float(s_stop)
        self.headroom = headroom
        self.group = group
        self.dev = scene.device
        self.n = len(scene)
        self.lib = _lib.lib()
        self.sd = _scene_desc(scene)
        n, dev = self.n, self.dev
        shapes = {(v.n_rg, v.n_az) for v in self.views}
        if len(shapes) != 1:
            raise ValueError("all views of a step must share the image size")
        # the slot buffers (tile grid, ranges, work items, splat scratch) are
        # sized from views[0]: every view must have the same ray grid
        if len({(v.n_u, v.n_v) for v in self.views}) != 1:
            raise ValueError("all views of a step must share the computation-plane ray grid")
        self.img_shape = shapes.pop()
        # geometry epilogue batches: `geo_batch` views' projections, partial
        # records and imaging-plane sums stay resident until one batched
        # sdgr_grad_geometry_batch call consumes them
        max_batch = int(self.lib.sdgr_max_batch())
        self.geo_batch = max(1, min(int(geo_batch or max_batch), max_batch, len(self.views)))
        # batch sizes of a step: uniform by default; `ramp` r > 0 gives a
        # geometric ramp (r, 3r, 9r, ... capped) that starts the first walks
        # after an r-view preprocessing pass (profiles/timeline.py: 1.5 ms
        # instead of 4.3 ms into the c4 step) -- measured 1194 vs 1220
        # views/s: the step is throughput-bound, the shorter fill only moves
        # the preprocessing under the walks (profiles/ROUND2.md)
        self.batches = self._schedule(len(self.views), self.geo_batch, ramp)
        # lanes: views alternate between `lanes` streams, each with its own
        # per-view working buffers, so one view's latency-bound walks overlap
        # another view's preprocessing; the batch's geometry joins the lanes
        self.n_lanes = max(1, min(int(lanes), self.geo_batch))
        self.lanes = [self._lane() for _ in range(self.n_lanes)]
        # the batched preprocessing (K1-K5 of a whole batch) runs on its own
        # stream, one batch ahead of the lanes' walks
        self.pre_stream = torch.cuda.Stream(device=dev)
        # training mode: each view's dL/dS comes from the device loss against
        # its target image (optimize.loss), written into the run's dlds buffer
        self.targets = None
        if targets is not None:
            if tuple(targets.shape) != (len(self.views),) + self.img_shape:
                raise ValueError("targets must be (V, n_range, n_azimuth)")
            from .train import LossBuffers
            self.targets = targets.to(device=dev, dtype=torch.float64).contiguous()
            self.lambda_ssim, self.max_val = float(lambda_ssim), float(max_val)
            self.loss_values = torch.zeros((len(self.views),), dtype=torch.float64, device=dev)
            for ln in self.lanes:
                ln.loss = LossBuffers(*self.img_shape, device=dev)
        # two slot sets: batch b's geometry overlaps batch b+1's views
        self.n_slots = 2 * self.geo_batch if len(self.views) > self.geo_batch else self.geo_batch
        self.proj_bufs = [self._projection_bufs() for k in range(self.n_slots)]
        self.pds = [pd for pd, _ in self.proj_bufs]
        self.pd = self.pds[0]
        self.counters, self.member_pairs = self.proj_bufs[0][1]["counters"], self.proj_bufs[0][1]["member_pairs"]
        self.order = _empty((n,), torch.int32, dev)
        self.acc_imgs = [_empty((6, n), torch.float64, dev) for _ in range(self.n_slots)]
        self.acc_img = self.acc_imgs[0]
        self.status = torch.zeros((4,), dtype=torch.int32, device=dev)
        # one device word per step: != 0 when any pair / replay buffer overflowed
        # (the step's gradients are then truncated); guards the Adam update
        self.overflow = torch.zeros((), dtype=torch.int32, device=dev)
        self.generation = 0   # bumped by every (re)allocation: captured graphs are stale
        # gradients: one flat float32 buffer so the all-reduce is one call
        self.grads = self._grad_views()
        self.gd = self.grads.desc()
        self.cap = None
        self.planes = None
        self.stage_events = None
        self.graph = None
        self.graph_launches = 0

    @staticmethod
    def _schedule(n_views: int, cap: int, ramp: int | None) -> list:
        """Views per batch: ramp, 3 ramp, 9 ramp, ... capped at `cap`
        (ramp = 0 or >= cap: uniform batches of `cap`)."""
        if ramp is None:
            ramp = int(os.environ.get("SDGR_BATCH_RAMP", "0"))
        if n_views <= cap:
            return [n_views]         # one batch: nothing to overlap its preprocessing with
        out, left, b = [], n_views, (ramp if 0 < ramp < cap else cap)
        while left > 0:
            k = min(b, cap, left)
            out.append(k)
            left -= k
            b = min(cap, 3 * b)
        return out

    # -- buffers ------------------------------------------------------------
    class _Lane:
        pass

    def _lane(self):
        """Stream + per-view working buffers of one lane (pair buffers are
        added by _alloc_planes once the capacities are known)."""
        n, dev = self.n, self.dev
        ln = MultiViewStep._Lane()
        ln.stream = torch.cuda.Stream(device=dev)
        ln.intensity = _empty((n,), torch.float64, dev)
        ln.image = _empty(self.img_shape, torch.float64, dev)
        return ln

    def _projection_bufs(self):
        """One set of per-view projection records (K1 outputs) + its descriptor."""
        n, dev = self.n, self.dev
        rec = {}
        pd = _lib.ProjectionDesc()
        pd.n = n
        for name in ("comp", "img"):
            pl = _lib.Plane()
            r = dict(inv_cov=_empty((n, 4), torch.float64, dev), n_tiles=_empty((n,), torch.int32, dev))
            if name == "comp":
                # 64-byte rows the pair-record gather reads, 16-byte rows the
                # fused count + emit reads; the SoA uv / bbox / masks they
                # replace are neither allocated nor written
                r["packed"] = _empty((n, 8), torch.float64, dev)
                r["emit"] = _empty((n, 2), torch.int64, dev)
                pl.packed, pl.emit = ptr(r["packed"]), ptr(r["emit"])
            else:
                r.update(uv=_empty((n, 2), torch.float64, dev), bbox=_empty((n, 4), torch.int16, dev),
                         cell_mask=_empty((n,), torch.int64, dev), tile_mask=_empty((n,), torch.int64, dev))
                pl.uv, pl.bbox = ptr(r["uv"]), ptr(r["bbox"])
                pl.cell_mask, pl.tile_mask = ptr(r["cell_mask"]), ptr(r["tile_mask"])
            pl.inv_cov, pl.n_tiles, pl.cov = ptr(r["inv_cov"]), ptr(r["n_tiles"]), None
            rec[name] = r
            setattr(pd, name, pl)
        for k, dt in (("depth_key", torch.int64), ("phase_raw", torch.float64), ("flags", torch.uint8)):
            rec[k] = _empty((n,), dt, dev)
            setattr(pd, k, ptr(rec[k]))
        pd.kappa = pd.phase = None   # carried by the packed rows
        rec["counters"] = torch.zeros((4,), dtype=torch.int32, device=dev)
        rec["member_pairs"] = torch.zeros((2,), dtype=torch.int64, device=dev)
        pd.counters, pd.member_pairs = ptr(rec["counters"]), ptr(rec["member_pairs"])
        pd.ke_act = None
        pd.look = None
        return pd, rec

    def _grad_views(self) -> SceneGradients:
        # SoA views into one flat buffer keep each group contiguous and make
        # the all-reduce one call
        self.flat_soa = torch.zeros((GRAD_WIDTH * self.n,), dtype=torch.float32, device=self.dev)
        return grad_views(self.flat_soa, self.n)

    def _alloc_planes(self, cap_pairs: dict):
        n, dev = self.n, self.dev
        v = self.views[0]
        cap = cap_pairs[0]
        nu, nv = v.n_u, v.n_v
        tx, ty = -(-nu // TILE), -(-nv // TILE)
        # depth segments: a lone view wants ~32 per SM so its walk has no tail
        # (_seg_len); with 8 views in flight the tails overlap, and longer
        # segments mean fewer pass-A items and segment scans: 2048 measured
        # +3 % views/s at c4 over 512 (profiles/ROUND1.md)
        seg = _seg_len(cap) if os.environ.get("SDGR_SEG_LEN") else max(_seg_len(cap), MULTIVIEW_SEG_LEN)
        max_items = -(-cap // seg) + tx * ty
        # per slot: the binning outputs a view's walks and geometry read (the
        # batched preprocessing of batch b+1 fills one slot set while batch b's
        # lanes walk the other); only the computation plane is binned -- the
        # splat is Gaussian-parallel
        self.slot_t, self.slot_tiles, self.slot_order, self.slot_offsets = [], [], [], []
        for _ in range(self.n_slots):
            t = dict(
                pair_tile=_empty((cap,), torch.int32, dev), pair_pos=_empty((cap,), torch.int32, dev),
                pair_prim=_empty((cap,), torch.int32, dev), pre_prim=_empty((cap,), torch.int32, dev),
                pair_start=_empty((n,), torch.int32, dev), tile_range=_empty((tx * ty, 2), torch.int32, dev),
                items=_empty((max_items, 4), torch.int32, dev), tile_first=_empty((tx * ty,), torch.int32, dev),
                n_items=torch.zeros((4,), dtype=torch.int32, device=dev),
                pair_rec=_empty((cap, _lib.PAIR_REC_BYTES), torch.uint8, dev),
            )
            d = _lib.TilesDesc()
            d.plane, d.tiles_x, d.tiles_y, d.n_tiles = 0, tx, ty, tx * ty
            d.n_pairs = cap
            for k in ("pair_tile", "pair_pos", "pair_prim", "pre_prim", "pair_start", "tile_range", "items",
                      "tile_first", "n_items", "pair_rec"):
                setattr(d, k, ptr(t[k]))
            d.seg_len, d.max_items, d.device_count = seg, max_items, 1
            self.slot_t.append(t)
            self.slot_tiles.append(d)
            self.slot_order.append(_empty((n,), torch.int32, dev))
            self.slot_offsets.append(_empty((n + 1,), torch.int32, dev))
        # one batch workspace: the preprocessing runs on one stream
        self.ws_bytes = self.lib.sdgr_batch_workspace_bytes(n, cap, self.geo_batch)
        self.ws = _empty((self.ws_bytes,), torch.uint8, dev)
        # per lane: the walks' scratch (segment sums, partial intensities, replay log)
        for ln in self.lanes:
            ln.t = dict(
                seg_a=_empty((max_items * 256,), torch.float64, dev),
                seg_b=_empty((max_items * 256,), torch.float64, dev),
                seg_c=_empty((max_items * 256,), torch.float64, dev),
                partial_I=_empty((cap,), torch.float64, dev),
            )
            ln.splat_scratch = _empty((v.n_rg * v.n_az + 1,), torch.int64, dev)
            # live-pair log: member pairs bound every view's live pairs
            ln.replay = ReplayLog(int(getattr(self, "calib_tc", cap * 16) * self.headroom), max_items, seg, dev, cap)
        ln0 = self.lanes[0]
        self.replay = ln0.replay
        self.intensity, self.image, self.splat_scratch = ln0.intensity, ln0.image, ln0.splat_scratch
        self.slot_partial = [_empty((cap, 8), torch.float64, dev) for _ in range(self.n_slots)]
        self.cap = dict(cap_pairs)
        # graphs captured before point at the freed buffers
        self.graph = None
        self.generation += 1

    def calibrate(self):
        """Measure the pair counts of every view (host syncs) and size buffers."""
        mx = {0: 1, 1: 1}
        st = _stream()
        ws_bytes = self.lib.sdgr_workspace_bytes(self.n, 1)
        ws = _empty((ws_bytes,), torch.uint8, self.dev)
        off = {pl: _empty((self.n + 1,), torch.int32, self.dev) for pl in (0, 1)}
        self.calib_t16 = []
        self.calib_tc_all = []
        for v in self.views:
            _check(self.lib.sdgr_project(C.byref(self.sd), C.byref(v), C.byref(self.pd), st), "sdgr_project")
            _check(self.lib.sdgr_depth_order(C.byref(self.pd), ptr(self.order), ptr(ws), ws_bytes, st),
                   "sdgr_depth_order")
            for pl in (0, 1):
                _check(self.lib.sdgr_count_pairs(C.byref(self.pd), pl, ptr(self.order) if pl == 0 else None,
                                                 ptr(off[pl]), ptr(ws), ws_bytes, st), "sdgr_count_pairs")
            tot = torch.cat([torch.stack([off[0][self.n], off[1][self.n]]).to(torch.int64),
                             self.member_pairs]).cpu().tolist()
            self.calib_tc = max(getattr(self, "calib_tc", 0), tot[2])
            self.calib_tc_all.append(tot[2])
            tot = tot[:2]
            mx = {0: max(mx[0], tot[0]), 1: max(mx[1], tot[1])}
            self.calib_t16.append(tot)
        self.calib_t16_mean = {pl: float(np.mean([t[pl] for t in self.calib_t16])) for pl in (0, 1)}
        self.calib_tc_mean = float(np.mean(self.calib_tc_all))
        self._alloc_planes({pl: int(mx[pl] * self.headroom) + 1024 for pl in (0, 1)})
        return mx

    # -- one view -----------------------------------------------------------
    def _preprocess(self, views, s0: int, ev=None):
        """K1-K5 of a batch of views into slots s0..s0+len(views)-1, each stage
        one launch over the whole batch (sdgr_*_batch), on the current stream."""
        lib, st, k = self.lib, _stream(), len(views)
        Views, Projs, Tiles, Ptrs = _lib.View * k, _lib.ProjectionDesc * k, _lib.TilesDesc * k, C.c_void_p * k
        vs, pds = Views(*views), Projs(*self.pds[s0:s0 + k])
        orders = Ptrs(*[ptr(o) for o in self.slot_order[s0:s0 + k]])
        offsets = Ptrs(*[ptr(o) for o in self.slot_offsets[s0:s0 + k]])
        tiles = Tiles(*self.slot_tiles[s0:s0 + k])

        def mark(i):
            if ev is not None:
                ev[i].record()
        mark(0)
        _check(lib.sdgr_project_batch(C.byref(self.sd), k, vs, pds, st), "sdgr_project_batch")
        mark(1)
        _check(lib.sdgr_depth_order_batch(k, pds, orders, ptr(self.ws), self.ws_bytes, st), "sdgr_depth_order_batch")
        mark(2)
        _check(lib.sdgr_bin_batch(k, pds, vs, 0, orders, offsets, tiles, ptr(self.ws), self.ws_bytes, st),
               "sdgr_bin_batch")
        mark(3)

    def _view(self, v, dlds: torch.Tensor, slot: int, ev=None, ln=None, vi: int = 0):
        """K6-K9 of one view held in batch slot `slot` (preprocessed by
        _preprocess; the geometry epilogue runs per batch), on the current
        stream with lane `ln`'s walk scratch."""
        lib, st = self.lib, _stream()
        ln = ln if ln is not None else self._lane_of(slot)
        pd = C.byref(self.pds[slot])
        t0 = ln.t
        tiles = C.byref(self.slot_tiles[slot])
        acc = self.acc_imgs[slot]

        def mark(i):
            if ev is not None:
                ev[i].record()
        mark(0)
        _check(lib.sdgr_composite_forward(C.byref(v), pd, tiles, self.s_stop, ptr(t0["seg_a"]),
                                          ptr(t0["seg_b"]), ptr(t0["partial_I"]), ptr(ln.intensity),
                                          ptr(self.status), C.byref(ln.replay.desc_c), st),
               "sdgr_composite_forward")
        mark(1)
        _check(lib.sdgr_splat(C.byref(v), pd, ptr(ln.intensity), ptr(ln.splat_scratch), ptr(ln.image), st),
               "sdgr_splat")
        if self.targets is not None:   # dL/dS of this view from the device loss
            h, w = self.img_shape
            _check(lib.sdgr_loss(ptr(ln.image), ptr(self.targets[vi]), h, w, self.lambda_ssim, self.max_val,
                                 C.cast(ln.loss.kernel, C.c_void_p), ptr(self.loss_values[vi]), ptr(dlds),
                                 ptr(ln.loss.scratch), st), "sdgr_loss")
        mark(2)
        _check(lib.sdgr_grad_image(C.byref(v), pd, ptr(ln.intensity), ptr(dlds), ptr(acc), st),
               "sdgr_grad_image")
        mark(3)
        # seg_b holds the forward's exclusive prefixes; seg_a is reused as scratch
        _check(lib.sdgr_grad_intensity(C.byref(v), pd, tiles, self.s_stop, ptr(t0["seg_b"]),
                                       ptr(acc[0]), ptr(t0["seg_a"]), ptr(t0["seg_c"]),
                                       ptr(self.slot_partial[slot]), C.byref(ln.replay.desc_c), st),
               "sdgr_grad_intensity")
        mark(4)

    def _lane_of(self, slot: int, n_lanes: int | None = None):
        return self.lanes[(slot % self.geo_batch) % (n_lanes or self.n_lanes)]

    def _geometry(self, views, s0: int = 0, ev=None):
        """Batched K10 over the views held in slots s0..s0+len(views)-1."""
        k = len(views)
        Views = _lib.View * k
        Projs = _lib.ProjectionDesc * k
        Tiles = _lib.TilesDesc * k
        Ptrs = C.c_void_p * k
        if ev is not None:
            ev[0].record()
        _check(self.lib.sdgr_grad_geometry_batch(
            C.byref(self.sd), k, Views(*views), Projs(*self.pds[s0:s0 + k]), Tiles(*self.slot_tiles[s0:s0 + k]),
            Ptrs(*[ptr(a) for a in self.acc_imgs[s0:s0 + k]]), Ptrs(*[ptr(p) for p in self.slot_partial[s0:s0 + k]]),
            C.byref(self.gd), 1, _stream()), "sdgr_grad_geometry_batch")
        if ev is not None:
            ev[1].record()

    def run(self, dlds: torch.Tensor, timing: bool = False, check: bool = True, stats: list | None = None,
            allreduce: bool = True, lanes: int | None = None):
        """Forward + backward of every view; dlds: (V, H, W) float64 on device.
        Returns the accumulated SceneGradients (all-reduced if distributed).
        stats: if a list, one device tensor per view is appended holding
        (live pairs logged by the forward, work items) -- no host sync.
        lanes: use only the first `lanes` view streams (default: all)."""
        if self.cap is None:
            self.calibrate()
        if dlds.shape[0] != len(self.views):
            raise ValueError("one upstream image gradient per view")
        self.flat_soa.zero_()
        self.status.zero_()
        for t in self.slot_t:
            t["n_items"].zero_()        # sticky overflow flags: one check per step
        for ln in self.lanes:
            ln.replay.cursor.zero_()
        evs, pevs, gevs = [], [], []
        B = self.geo_batch
        n_sets = self.n_slots // B
        main = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(main)             # lanes start after the zeroing above
        L = max(1, min(int(lanes or self.n_lanes), self.n_lanes))
        active = self.lanes[:L]
        # one lane = fully serial (each kernel alone on the GPU: the
        # single-stream timing mode), preprocessing included
        pre = active[0].stream if L == 1 else self.pre_stream
        for s_ in set([pre] + [ln.stream for ln in active]):
            s_.wait_event(start)
        geo_done = [None] * n_sets     # geometry that last read each slot set
        geo_last = None
        starts = np.cumsum([0] + self.batches[:-1]).tolist()
        for bi, (b0, nb) in enumerate(zip(starts, self.batches)):
            batch = self.views[b0:b0 + nb]
            s0 = (bi % n_sets) * B
            wait_geo = geo_last if L == 1 else geo_done[bi % n_sets]
            if wait_geo is not None:
                pre.wait_event(wait_geo)   # the slot set's previous geometry has read it
            with torch.cuda.stream(pre):
                pev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if timing else None
                self._preprocess(batch, s0, pev)
                ready = torch.cuda.Event()
                ready.record(pre)
            if timing:
                pevs.append(pev)
            for ln in active:
                ln.stream.wait_event(ready)
            for k, v in enumerate(batch):
                ln = self._lane_of(s0 + k, L)
                with torch.cuda.stream(ln.stream):
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if timing else None
                    self._view(v, dlds[b0 + k], s0 + k, ev, ln, vi=b0 + k)
                    if stats is not None:
                        stats.append(torch.stack([ln.replay.cursor[0],
                                                  self.slot_t[s0 + k]["n_items"][0].to(torch.int64)]))
                if timing:
                    evs.append(ev)
            for ln in active:          # this batch's views are done (lanes run on)
                main.wait_stream(ln.stream)
            gev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if timing else None
            self._geometry(batch, s0, gev)
            done = torch.cuda.Event()
            done.record(main)
            geo_done[bi % n_sets] = done
            geo_last = done
            if timing:
                gevs.append(gev)
        main.wait_stream(pre)
        # fold every overflow flag into one word (device ops: graph-capturable)
        flags = [t["n_items"][1] for t in self.slot_t] + [ln.replay.cursor[1].to(torch.int32) for ln in self.lanes]
        torch.amax(torch.stack(flags), dim=0, out=self.overflow)
        self.stage_events = (evs, pevs, gevs)
        if allreduce and (self.group is not None or
                          (torch.distributed.is_available() and torch.distributed.is_initialized())):
            self.allreduce()
        if check:
            self.check()
        return self.grads

    # -- CUDA graph of a whole step -------------------------------------------
    def capture(self, dlds: torch.Tensor, warm: bool = True, lanes: int | None = None):
        """Record one step (every view's forward + backward; no all-reduce, no
        host check) as a CUDA graph over static buffers: the scene tensors and
        `dlds` are read where they live, so callers overwrite them in place and
        call graph_step().  Kernel launches are replayed without host work or
        per-launch gaps.  Returns the number of library kernels in the graph."""
        if self.cap is None:
            self.calibrate()
        if warm:
            self.run(dlds, check=False, lanes=lanes)   # first-call attributes / occupancy queries
        torch.cuda.synchronize()
        n0 = self.lib.sdgr_launch_count()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.run(dlds, check=False, allreduce=False, lanes=lanes)
        self.graph_launches = int(self.lib.sdgr_launch_count() - n0)
        return self.graph_launches

    def graph_step(self, check: bool = False):
        """One captured step (+ the all-reduce when distributed)."""
        if self.graph is None:
            raise StateError("no captured graph (calibrate() reallocates the buffers): call capture() again")
        self.graph.replay()
        if self.group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()):
            self.allreduce()
        if check:
            self.check()
        return self.grads

    def allreduce(self):
        allreduce_grads(self.flat_soa, self.n, self.group)

    def bind(self, scene: DeviceScene, flat_soa: torch.Tensor | None = None):
        """Point the step at another scene of the same size (and optionally
        another flat gradient buffer).  A graph captured afterwards reads and
        writes those buffers; graphs captured before keep theirs."""
        if len(scene) != self.n or scene.dtype != self.scene.dtype:
            raise ValueError("bind: scene must match the step's size and dtype")
        self.scene, self.sd = scene, _scene_desc(scene)
        if flat_soa is not None:
            if flat_soa.shape != self.flat_soa.shape or flat_soa.dtype != torch.float32:
                raise ValueError("bind: flat gradient buffer shape/dtype mismatch")
            self.flat_soa = flat_soa
            self.grads = grad_views(flat_soa, self.n)
            self.gd = self.grads.desc()

    def check(self):
        """One host read per step: capacity overflow and non-finite status."""
        bad, ov = torch.stack([self.status[0], self.overflow]).cpu().tolist()
        if ov:
            raise OverflowError("pair capacity exceeded; recalibrate")
        if bad:
            raise NumericalError("non-finite intensity in a multi-view step")

    def stage_times_ms(self):
        """Per-stage device time summed over the last timed run's views
        (project / depth_sort / binning: the batched launches; grad_geometry:
        summed over its batched launches)."""
        pre_names = ("project", "depth_sort", "binning")
        names = ("forward_comp", "splat", "grad_image", "grad_intensity")
        out = dict.fromkeys(pre_names + names + ("grad_geometry",), 0.0)
        evs, pevs, gevs = self.stage_events or ([], [], [])
        for ev in pevs:
            for i, nm in enumerate(pre_names):
                out[nm] += ev[i].elapsed_time(ev[i + 1])
        for ev in evs:
            for i, nm in enumerate(names):
                out[nm] += ev[i].elapsed_time(ev[i + 1])
        for ev in gevs:
            out["grad_geometry"] += ev[0].elapsed_time(ev[1])
        return out


class HostStepPipeline:
    """Steps fed from and returned to pinned host memory, pipelined.

    Each submit() takes one step's inputs in host memory -- the scene arrays
    and the per-view dL/dS -- and delivers that step's accumulated gradients
    (the flat (30 n,) float32 SoA of MultiViewStep) back into a host buffer.
    Two device banks (scene, dL/dS, gradients) alternate: step k+1's uploads
    run on a copy stream while step k's graph computes, and step k's gradient
    download overlaps step k+1's compute, so the PCIe copies hide under the
    kernels.  Every step still moves all of its inputs and its result.

    This is the host-facing shape of the reference's loop: per step the host
    hands over parameters and upstream gradients and reads the parameter
    gradients back (optimize.py:395-425 around render/backward).
    """

    def __init__(self, step: MultiViewStep, dl_dtype=torch.float32):
        if step.cap is None:
            step.calibrate()
        self.step = step
        dev, n = step.dev, step.n
        V = len(step.views)
        shape = (V,) + step.img_shape
        base_scene, base_flat = step.scene, step.flat_soa
        self.banks = []
        for b in range(2):
            scene = base_scene if b == 0 else DeviceScene(*(a.clone() for a in base_scene.arrays()))  # valid warm-up input
            flat = base_flat if b == 0 else torch.zeros_like(base_flat)
            dl_in = torch.empty(shape, dtype=dl_dtype, device=dev)
            dl64 = dl_in if dl_dtype == torch.float64 else torch.empty(shape, dtype=torch.float64, device=dev)
            self.banks.append(dict(scene=scene, flat=flat, dl_in=dl_in, dl64=dl64, graph=None,
                                   uploaded=torch.cuda.Event(), computed=torch.cuda.Event(),
                                   downloaded=torch.cuda.Event(), used=False))
        self.up = torch.cuda.Stream(device=dev)
        self.down = torch.cuda.Stream(device=dev)
        self.k = 0
        self.launches = 0
        for bk in self.banks:
            step.bind(bk["scene"], bk["flat"])
            step.run(bk["dl64"].zero_(), check=False, allreduce=False)   # warm: attributes, occupancy queries
            torch.cuda.synchronize()
            n0 = step.lib.sdgr_launch_count()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                if bk["dl64"] is not bk["dl_in"]:
                    bk["dl64"].copy_(bk["dl_in"])
                step.run(bk["dl64"], check=False, allreduce=False)
            bk["graph"] = g
            self.launches = int(step.lib.sdgr_launch_count() - n0)
        step.bind(base_scene, base_flat)
        self.generation = step.generation

    def submit(self, host_scene: dict, host_dl: torch.Tensor, host_out: torch.Tensor):
        """Queue one step.  host_scene: {group: pinned tensor} for positions,
        rotations, log_scales, sh_coeffs, ke_raw; host_dl: pinned (V, H, W);
        host_out: pinned float32 (30 n,) receiving the gradients.  Returns an
        event that completes when host_out holds this step's result."""
        if self.step.generation != self.generation:
            raise StateError("the step was recalibrated after this pipeline captured it; build a new pipeline")
        bk = self.banks[self.k % 2]
        self.k += 1
        main = torch.cuda.current_stream()
        with torch.cuda.stream(self.up):
            if bk["used"]:
                self.up.wait_event(bk["computed"])      # the bank's previous graph has read its inputs
            for g, dst in zip(("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw"),
                              bk["scene"].arrays()):
                dst.copy_(host_scene[g], non_blocking=True)
            bk["dl_in"].copy_(host_dl, non_blocking=True)
            bk["uploaded"].record(self.up)
        main.wait_event(bk["uploaded"])
        if bk["used"]:
            main.wait_event(bk["downloaded"])            # its previous gradients have left the device
        bk["graph"].replay()
        if self.step.group is not None or (torch.distributed.is_available() and torch.distributed.is_initialized()):
            allreduce_grads(bk["flat"], self.step.n, self.step.group)
        bk["computed"].record(main)
        with torch.cuda.stream(self.down):
            self.down.wait_event(bk["computed"])
            host_out.copy_(bk["flat"], non_blocking=True)
            bk["downloaded"].record(self.down)
        bk["used"] = True
        done = torch.cuda.Event()
        done.record(self.down)
        return done

    def drain(self):
        """Make the current stream wait for every queued download."""
        torch.cuda.current_stream().wait_stream(self.down)

    def check(self):
        self.step.check()
