#!/usr/bin/env python
"""SDGR benchmark: SAR views/s, forward + custom backward, 1M Gaussians at 512x512.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl sdgr|reference]

Workload (BASELINE.json configs[3] / SURVEY.md §8d c4): 16 tanks on a 4x4
grid (20 m pitch), 1 000 000 Gaussians, 512x512 views at az 0:360:3 x el
{30, 45, 60} (360 views).  A step = every rank renders and back-propagates
its shard of `--views-per-rank` views (default 45, so 8 ranks cover all 360)
with gradients accumulated on the device, then one NCCL all-reduce of the
per-Gaussian gradients.  Weak scaling: per-GPU work is fixed as N grows.

`value`  : views/s over all ranks, inputs resident in HBM, CUDA events, max
           over ranks.
`e2e`    : the same step through the public API from pinned host memory
           (scene + upstream gradients H2D, accumulated gradients D2H).
`roofline`: the dominant kernel (largest device time in an instrumented
           single-stream step), timed with CUDA event nodes around each of
           its launches in a single-stream graph replay of the same step run
           just before the timed region (sdgr_profile_begin/end; in the
           concurrent step a launch's events would also span its wait for SM
           slots held by the other lanes); achieved = its algorithmic HBM
           bytes per launch (kernel_bytes()) / mean launch
           time; traffic = ncu DRAM bytes per launch from profiles/
           (committed capture) when present.
`cpu_baseline`: the oracle port (oracle/sdgr_oracle.py, the reference's
           algorithm restated in NumPy + C) on the host cores, rank 0, N=1.
`--impl reference`: the reference's CPU path (oracle port; the reference is
           pure Python and cannot travel to the GPU box) on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SAR views/sec fwd+bwd (1M Gaussians, 512² px) at 1/2/4/8 B200; % HBM roofline"
UNIT = "views/s"
RSS_PER_ORACLE_PROC = 6.0e9   # bytes, oracle fwd+bwd at 1M Gaussians / 512^2 (measured 4.9 GB peak)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sdgr", choices=("sdgr", "reference"))
    ap.add_argument("--workload", default="c4", choices=tuple(WORKLOADS),
                    help="SURVEY.md §8d configuration (default c4, the metric's configuration)")
    ap.add_argument("--n", type=int, default=None, help="override the workload's Gaussian count")
    ap.add_argument("--size", type=int, default=None, help="override the workload's image size")
    ap.add_argument("--sigma", type=float, default=None, help="isotropic Gaussian scale in m (c5 sweep)")
    ap.add_argument("--scene-order", default="morton", choices=("morton", "native", "random"),
                    help="memory order of the synthetic scene's Gaussians (make_scene)")
    ap.add_argument("--views-per-rank", type=int, default=None)
    ap.add_argument("--dropin-views", type=int, default=10,
                    help="views timed through render_forward + backward with host arrays (0 = skip)")
    ap.add_argument("--param-dtype", default="f32", choices=("f32", "f64"))
    ap.add_argument("--s-stop", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-procs", type=int, default=0)
    ap.add_argument("--lanes", type=int, default=8, help="concurrent view streams per GPU")
    ap.add_argument("--geo-batch", type=int, default=None, help="views per batched launch (default: the build's max)")
    ap.add_argument("--dist-backend", default="nccl", choices=("nccl", "gloo"),
                    help="gloo + --share-gpu: exercise the N>1 code path with every rank on cuda:0 "
                         "(a functional check, never a scaling number)")
    ap.add_argument("--share-gpu", action="store_true", help="all ranks on cuda:0 (functional check only)")
    a = ap.parse_args()
    w = WORKLOADS[a.workload]
    a.n = a.n or w["n"]
    a.size = a.size or w["size"]
    a.views_per_rank = a.views_per_rank or w["views_per_rank"]
    return a


# SURVEY.md §8d configurations (BASELINE.json configs[1..4]); the metric is quoted on c4
WORKLOADS = {
    "c2": dict(n=100_000, size=256, views_per_rank=36, scene="tank", az=range(0, 360, 10), el=(45.0,),
               label="single vehicle (tank_preset), {n} Gaussians, {size}x{size}, az 0:360:10 x el 45"),
    "c3": dict(n=300_000, size=256, views_per_rank=72, scene="tank", az=range(0, 360, 15), el=(15.0, 45.0, 75.0),
               label="single vehicle (tank_preset), {n} Gaussians, {size}x{size}, az 0:360:15 x el 15/45/75"),
    "c4": dict(n=1_000_000, size=512, views_per_rank=45, scene="grid", az=range(0, 360, 3), el=(30.0, 45.0, 60.0),
               label="16-tank grid (20 m pitch), {n} Gaussians, {size}x{size}, az 0:360:3 x el 30/45/60"),
    "c5": dict(n=1_000_000, size=512, views_per_rank=8, scene="grid", az=range(0, 360, 45), el=(45.0,),
               label="backward stress: 16-tank grid, {n} Gaussians, isotropic sigma {sigma} m, {size}x{size}, el 45"),
}


def workload_label(args) -> str:
    return f"{args.workload}: " + WORKLOADS[args.workload]["label"].format(n=args.n, size=args.size,
                                                                          sigma=args.sigma)


def view_list(size: int, workload: str = "c4"):
    from paper_2506_21633_b200.radar import RadarConfig
    w = WORKLOADS[workload]
    out = []
    for az in w["az"]:
        for el in w["el"]:
            out.append(RadarConfig(azimuth_deg=float(az), elevation_deg=el, altitude_m=0.5, range_res_m=0.3,
                                   azimuth_res_m=0.3, n_range=size, n_azimuth=size))
    return out


def make_scene(n: int, workload: str = "c4", sigma: float | None = None, order: str = "morton"):
    """The workload's synthetic scene.  order: "morton" (default) stores the
    Gaussians in spatial_order (the framework's recommended layout, applied
    once here, outside any timed region); "native" keeps the sampler's
    per-face order; "random" shuffles (the worst case)."""
    from paper_2506_21633_b200 import targets
    from paper_2506_21633_b200.scene import spatial_sort
    if WORKLOADS[workload]["scene"] == "tank":   # budgets 0.6 / 0.3 / 0.1 as SURVEY §8d c2 / c3
        b = [int(round(0.6 * n)), int(round(0.3 * n))]
        scene = targets.composite_target(targets.tank_preset(), b + [n - sum(b)], seed=3)
    else:
        scene = targets.tank_grid(n_total=n)
    if sigma is not None:
        scene.log_scales[:] = np.log(sigma)
    if order == "morton":
        scene = spatial_sort(scene)[0]
    elif order == "random":
        perm = np.random.default_rng(0).permutation(len(scene.positions))
        scene = type(scene)(*(getattr(scene, k)[perm] for k in
                              ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")))
    # float32-exact so the float32 device scene and the FP64 oracle see the same Gaussians
    return targets.to_float32_exact(scene)


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        self.tmp.flush()
        rows = []
        for line in Path(self.tmp.name).read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append((float(f[1]), float(f[2]), f[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = sorted(r[0] for r in rows)
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------- CPU side
_CPU_SCENE = None
_CPU_CFGS = None


def _oracle_warm(_):
    from oracle import sdgr_oracle as O
    O.oracle_exp(0.0)   # imports + C library load, no rendering
    return 0


def _oracle_view(i):
    from oracle import sdgr_oracle as O
    cfg = _CPU_CFGS[i % len(_CPU_CFGS)]
    rng = np.random.default_rng(i)
    t0 = time.perf_counter()
    f = O.render_forward(_CPU_SCENE, cfg)
    O.backward(f, rng.normal(size=f.image.shape))
    return time.perf_counter() - t0


def cpu_procs(requested: int = 0) -> int:
    cores = len(os.sched_getaffinity(0))
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 64e9
    by_ram = max(1, int(0.8 * avail // RSS_PER_ORACLE_PROC))
    p = min(cores, by_ram)
    return max(1, min(p, requested)) if requested else p


def cpu_run(scene, cfgs, procs: int, views: int):
    """Run `views` oracle fwd+bwd views on `procs` forked processes; returns wall s."""
    import multiprocessing as mp
    global _CPU_SCENE, _CPU_CFGS
    _CPU_SCENE, _CPU_CFGS = scene, cfgs
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_oracle_warm, range(procs))   # warm the workers (imports, C lib)
        t0 = time.perf_counter()
        pool.map(_oracle_view, range(views), chunksize=1)
        return time.perf_counter() - t0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import sdgr_oracle
    sdgr_oracle.build()
    scene = make_scene(args.n, args.workload, args.sigma, args.scene_order)
    cfgs = view_list(args.size, args.workload)
    procs = cpu_procs(args.cpu_procs)
    # warm-up: one-time costs only (fork, imports, page-in) on a small sample
    from paper_2506_21633_b200 import targets
    small = targets.to_float32_exact(targets.tank_grid(n_total=16_000))
    for _ in range(max(1, min(args.warmup, 1))):
        cpu_run(small, view_list(128), procs, procs)
    # each step renders + back-propagates one c4 view per process (~16 s); the
    # number of timed steps is capped so the arm ends within a few minutes
    # (the line reports the steps actually timed)
    times = [cpu_run(scene, cfgs, procs, procs)]
    budget_s = float(os.environ.get("SDGR_REF_BUDGET_S", "150"))
    steps_eff = max(1, min(args.steps, int(budget_s // max(times[0], 1e-3))))
    times += [cpu_run(scene, cfgs, procs, procs) for _ in range(steps_eff - 1)]
    ms = 1e3 * float(np.mean(times))
    value = procs / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(times), "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_label(args), "scene_order": args.scene_order,
                   "views_per_step": procs, "gaussians": args.n, "image": [args.size, args.size]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port", "cpu": cpu_model(),
                         "sample": f"{procs} {args.workload} views per step, one per forked process "
                                   "(oracle/sdgr_oracle.py: NumPy + C key chain, OPENBLAS_NUM_THREADS=1)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU side
SCENE_B = 12 + 16 + 12 + 64 + 8          # f32 positions, rotations, log_scales, sh_coeffs, ke_raw per Gaussian
GRAD_RMW_B = 2 * (29 * 4 + 4)            # f32 gradient groups + f32 visible count, read + written
PROJ_W_B = 2 * (16 + 32 + 8 + 8 + 8 + 4) + 8 * 4 + 1 + 64 + 16   # K1 outputs per Gaussian: two planes, key/kappa/phase/flags, packed + emit rows
REC_B = 80                               # packed computation-plane pair record
LOG_B = 8 + 8 + 8 + 1 + 1                # replay log entry: y1, t2, w, j, r


def kernel_bytes(kid: int, n: int, t16: float, live: float, items: float, batch: float) -> float:
    """Algorithmic HBM bytes of ONE launch of kernel `kid`:
    every input read once and every output written once, per view-level
    counts n (Gaussians), t16 (computation-plane pairs), live (logged live
    pairs), items (depth-segment work items); batch = views per batched
    launch (K1, binning and the geometry epilogue run once per batch)."""
    from paper_2506_21633_b200 import _lib as L
    if kid == L.K_PROJECT:     # parameters read once per batch, records written per view
        return n * SCENE_B + batch * n * PROJ_W_B
    if kid == L.K_SEGSUM:
        return REC_B * t16 + 8 * 256 * items
    if kid == L.K_WALK:
        return (REC_B + 8) * t16 + LOG_B * live + 8 * 256 * items
    if kid == L.K_REPLAY_GSUM:
        return (8 + 1 + 1) * live + (REC_B + 8 + 8) * t16 + 8 * 256 * items
    if kid == L.K_REPLAY_GRAD:
        return LOG_B * live + (REC_B + 8 + 64) * t16 + 2 * 8 * 256 * items
    if kid == L.K_GEOMETRY:
        per_view = n * (1 + 32 + 32 + 4 + 4 + 8 + 40) + 64 * t16
        return n * (SCENE_B + GRAD_RMW_B) + batch * per_view
    if kid == L.K_SPLAT:
        return n * (1 + 8 + 16 + 32 + 8 + 8)
    if kid == L.K_GRAD_IMAGE:
        return n * (1 + 8 + 16 + 32 + 8 + 8 + 48)
    if kid == L.K_GATHER:      # pos, pre, packed row + bbox, tile id read; record + prim written
        return batch * t16 * (4 + 4 + 64 + 8 + 4 + REC_B + 4)
    if kid == L.K_EMIT:        # order + 16 B emit row read, offsets / pair_start / key / value written
        return batch * (n * (4 + 16 + 4 + 4) + 8 * t16)
    if kid == L.K_ONESWEEP:    # 5 passes per batch: 3 over the N depth keys, 2 over the pairs (key + value r+w)
        return batch * 16 * (3 * n + 2 * t16) / 5
    return float("nan")


def preprocess_sort_roofline(n: int, step, stages: dict, views: int, peak: float) -> dict:
    """North-star target: preprocess + sort at >= 50 % of HBM
    roofline.  Algorithmic bytes per view by the survey's formula:
    B_pre = 184 N, B_rank = 192 N, B_bin = sum over planes of
    T16_p (12 + 24 ceil(b_p / 8) + 8), b_p = ceil(log2 tiles_p) + ceil(log2 N);
    time = the single-stream device time of the project + depth_sort +
    binning stages (each kernel alone on the GPU).  This design bins only the
    computation plane (the splat is Gaussian-parallel), so the formula's
    imaging-plane term is work it never does; `frac_comp_plane_only` drops it."""
    import math
    v0 = step.views[0]
    lg_n = math.ceil(math.log2(max(n, 2)))
    tiles = {0: -(-v0.n_u // 16) * -(-v0.n_v // 16), 1: -(-v0.n_az // 16) * -(-v0.n_rg // 16)}
    b_bin = {}
    for pl in (0, 1):
        bits = math.ceil(math.log2(max(tiles[pl], 2))) + lg_n
        b_bin[pl] = step.calib_t16_mean[pl] * (12 + 24 * math.ceil(bits / 8) + 8)
    b_pre, b_rank = 184.0 * n, 192.0 * n
    ms = (stages["project"] + stages["depth_sort"] + stages["binning"]) / views
    full = b_pre + b_rank + b_bin[0] + b_bin[1]
    comp = b_pre + b_rank + b_bin[0]
    return {"ms_per_view": ms, "bytes_per_view": full, "achieved_gbs": full / (ms / 1e3) / 1e9,
            "peak_gbs": peak, "frac": full / (ms / 1e3) / 1e9 / peak,
            "frac_comp_plane_only": comp / (ms / 1e3) / 1e9 / peak,
            "stages": ["project", "depth_sort", "binning"], "target_frac": 0.5,
            "formula": "SURVEY.md §8d: 184N + 192N + sum_p T16_p (12 + 24 ceil(b_p/8) + 8)"}


def _profile(lib):
    import ctypes as C
    from paper_2506_21633_b200 import _lib as L
    ms = (C.c_double * L.PROFILE_KERNELS)()
    cnt = (C.c_int64 * L.PROFILE_KERNELS)()
    if lib.sdgr_profile_end(ms, cnt) != 0:
        raise RuntimeError("sdgr_profile_end failed")
    return list(ms), list(cnt)


def ncu_traffic(kernel: str):
    """DRAM bytes per launch of `kernel` and its compute-side counters from
    the committed ncu capture summary (profiles/ncu_traffic.json)."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None, None, None
    d = json.loads(p.read_text())
    e = d.get("kernels", {}).get(kernel)
    return (e["dram_bytes_per_launch"], d.get("source"), e.get("compute")) if e else (None, None, None)


COMPOSITING = ("k_segsum", "k_walk<kContrib>", "k_replay<kGSum>", "k_replay<kGrad>")


def dropin_rate(sdgr, host_scene, cfgs, views: int, world: int, rank: int) -> dict:
    """Views/s of the reference-shaped call sequence -- one view per call, as
    the reference's optimize.train does (optimize.py:396-411):
    fwd = render_forward(numpy FP64 scene, config); grads = backward(fwd,
    numpy dL/dS) -> numpy FP64 SceneGradients.  Every call uploads the FP64
    scene (the caller's arrays, page-locked in place once they are seen
    again: direct DMA) and downloads FP64 gradients (DMA into recycled
    page-locked result blocks), so the rate is bounded by those copies;
    `copy_bound` times the same bytes as pinned <-> device DMA (the PCIe
    floor)."""
    import torch
    import torch.distributed as dist
    rng = np.random.default_rng(7 + rank)
    size = (cfgs[0].n_range, cfgs[0].n_azimuth)
    dls = [rng.normal(size=size) for _ in range(views)]
    # warm: first-call attributes, cached capacities, page-locking, result
    # blocks, and two passes over the timed view sequence so torch's caching
    # allocator has grown to its steady state (profiles/dropin_stalls.py: a
    # call that grows it can stall for tens to hundreds of ms)
    for i in range(max(5, 2 * views)):
        fwd = sdgr.render_forward(host_scene, cfgs[(i % views) % len(cfgs)])
        g = sdgr.backward(fwd, dls[i % views])
    torch.cuda.synchronize()
    import gc
    gc.collect()   # start the timed calls with a clean heap (a full collection inside costs 10-20 ms)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    call_ms = []   # host wall time per call (each call ends with its results on the host)
    for i in range(views):
        tc = time.perf_counter()
        fwd = sdgr.render_forward(host_scene, cfgs[i % len(cfgs)])
        g = sdgr.backward(fwd, dls[i])
        call_ms.append(1e3 * (time.perf_counter() - tc))
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1) / views
    # the bytes every call moves: FP64 scene + dL/dS up; image, FP64 gradients +
    # visible down.  The PCIe floor: the same bytes as DMA between pinned host
    # buffers and the device (a numpy caller additionally pays the host copies
    # between its pageable arrays and the pinned staging buffers)
    up = [getattr(host_scene, k) for k in ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")] + [dls[0]]
    down = list(g.param_arrays()) + [g.uv_grad_norm, g.visible, np.zeros(size)]
    h2d = sum(a.nbytes for a in up)
    d2h = sum(a.nbytes for a in down)
    hu = torch.empty((h2d,), dtype=torch.uint8, pin_memory=True)
    hd = torch.empty((d2h,), dtype=torch.uint8, pin_memory=True)
    du = torch.empty((h2d,), dtype=torch.uint8, device="cuda")
    dd = torch.empty((d2h,), dtype=torch.uint8, device="cuda")
    du.copy_(hu, non_blocking=True)
    hd.copy_(dd, non_blocking=True)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for _ in range(3):
        du.copy_(hu, non_blocking=True)
        hd.copy_(dd, non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    copy_ms = c0.elapsed_time(c1) / 3
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": world / (ms / 1e3), "unit": UNIT, "ms_per_view": ms, "wall_ms_per_view": 1e3 * wall / views,
            "median_call_ms": float(np.median(call_ms)), "call_ms": [round(x, 2) for x in call_ms],
            "views_timed": views, "h2d_bytes_per_view": int(h2d), "d2h_bytes_per_view": int(d2h),
            "copy_bound": {"ms_per_view": copy_ms, "views_per_s": world / (copy_ms / 1e3),
                           "what": "the same H2D + D2H bytes as pinned <-> device DMA (the PCIe floor)"},
            "call": "render_forward(numpy scene, cfg) + backward(fwd, numpy dL/dS) -> numpy FP64 gradients"}


def run_sdgr(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if args.share_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    import paper_2506_21633_b200 as sdgr
    from paper_2506_21633_b200.multiview import MultiViewStep

    pdt = torch.float32 if args.param_dtype == "f32" else torch.float64
    host_scene = make_scene(args.n, args.workload, args.sigma, args.scene_order)
    cfgs_all = view_list(args.size, args.workload)
    # rank r takes views r, r+W, ... and the first views_per_rank of them
    mine = [c for i, c in enumerate(cfgs_all) if i % world == rank]
    mine = (mine * (1 + args.views_per_rank // max(len(mine), 1)))[: args.views_per_rank]
    V = len(mine)
    # the reference-shaped drop-in first, in a process state like a user's
    # (before the multi-view step's buffers and pinned pipelines exist)
    dropin = None
    if args.dropin_views > 0:
        dropin = dropin_rate(sdgr, host_scene, mine, args.dropin_views, world, rank)
        torch.cuda.empty_cache()
    scene = sdgr.DeviceScene.from_host(host_scene, dtype=pdt)
    kw = {} if args.s_stop is None else {"s_stop": args.s_stop}
    step = MultiViewStep(scene, mine, lanes=args.lanes, geo_batch=args.geo_batch, **kw)
    totals = []
    mx = step.calibrate()
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    dl_host = torch.randn((V, args.size, args.size), generator=g, dtype=torch.float32)
    dlds = dl_host.to("cuda").double()

    def barrier():
        if world > 1:
            dist.barrier()

    from paper_2506_21633_b200 import _lib as L
    lib = L.lib()
    for _ in range(max(args.warmup, 3)):
        step.run(dlds)
    torch.cuda.synchronize()
    # one instrumented (untimed) single-stream step: per-kernel device time ->
    # the dominant kernel; per-view live pairs and work items for its bytes
    lib.sdgr_profile_begin(sum(1 << k for k in L.KERNEL_NAMES))
    vstats = []
    step.run(dlds, stats=vstats, lanes=1)
    prof_ms, prof_cnt = _profile(lib)
    st = torch.stack(vstats).double().mean(0).tolist()
    live_pv, items_pv = st[0], st[1]
    dom = max(L.KERNEL_NAMES, key=lambda k: prof_ms[k])
    # roofline timing: a single-stream graph of the step with event nodes
    # around the dominant kernel's launches.  (In the concurrent step below a
    # kernel's events also span the time its blocks wait for SM slots held by
    # other streams' kernels, so they would not be launch durations.)
    lib.sdgr_profile_begin(1 << dom)
    step.capture(dlds, warm=False, lanes=1)
    for _ in range(max(args.steps, 3)):
        step.graph_step()
    torch.cuda.synchronize()
    dom_ms, dom_cnt = _profile(lib)   # the last replay's launches of the dominant kernel
    # the timed step: one CUDA graph, views on `lanes` concurrent streams
    launches = step.capture(dlds, warm=False)
    step.graph_step()
    torch.cuda.synchronize()
    barrier()
    # ---------------- timed: inputs resident in HBM ----------------
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(args.steps):
            step.graph_step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
    step.check()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * V / (ms_max / 1e3)
    step.run(dlds, timing=True, check=False, lanes=1)   # untimed, graph-free, one stream: stage breakdown
    torch.cuda.synchronize()
    stages = step.stage_times_ms()

    # ---------------- e2e: public API from pinned host memory ----------------
    e2e = None
    if not args.no_e2e:
        from paper_2506_21633_b200.multiview import HostStepPipeline
        pin = {gname: torch.from_numpy(np.ascontiguousarray(getattr(host_scene, gname))).to(pdt).pin_memory()
               for gname in ("positions", "rotations", "log_scales", "sh_coeffs", "ke_raw")}
        dl_pin = dl_host.pin_memory()
        outs = [torch.empty(step.flat_soa.shape, dtype=torch.float32).pin_memory() for _ in range(2)]
        h2d = sum(p.numel() * p.element_size() for p in pin.values()) + dl_pin.numel() * dl_pin.element_size()
        d2h = outs[0].numel() * outs[0].element_size()
        # every step uploads its scene + dL/dS and downloads its gradients;
        # two device banks let step k's copies overlap steps k-1 / k+1
        pipe = HostStepPipeline(step, dl_dtype=dl_pin.dtype)
        for k in range(2):
            pipe.submit(pin, dl_pin, outs[k % 2])
        pipe.drain()
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        pipe.up.wait_event(f0)          # the first upload starts inside the timed region
        for k in range(args.steps):
            pipe.submit(pin, dl_pin, outs[k % 2])
        pipe.drain()
        f1.record()
        torch.cuda.synchronize()
        pipe.check()
        t = torch.tensor([f0.elapsed_time(f1) / args.steps], device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": world * V / (float(t.item()) / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(t.item()),
               "pipeline": "two device banks: step k's H2D/D2H overlap the neighbouring steps' compute"}

    # ---------------- e2e through the reference-shaped drop-in ----------------

    # ---------------- roofline: the dominant kernel ----------------
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    t16_pv = step.calib_t16_mean[0]
    batch = V / -(-V // step.geo_batch)
    launch_ms = dom_ms[dom] / max(dom_cnt[dom], 1)
    dom_per_step = dom_cnt[dom]
    bpl = kernel_bytes(dom, args.n, t16_pv, live_pv, items_pv, batch)
    achieved = bpl / (launch_ms / 1e3) / 1e9 if launch_ms > 0 else None
    traffic, traffic_src, dom_compute = ncu_traffic(L.KERNEL_NAMES[dom])
    step_ms_all = sum(prof_ms)
    # compute-side view of the compositing kernels: not HBM-shaped
    # work -- member / live pairs per second and the ncu pipe utilisation
    comp_ms = {nm: prof_ms[k] / V for k, nm in L.KERNEL_NAMES.items() if nm in COMPOSITING}
    compute_roofline = {
        "what": "compositing is latency / issue bound, not HBM bound: pairs per second and pipe utilisation",
        "member_pairs_per_view": float(step.calib_tc_mean) if hasattr(step, "calib_tc_mean") else None,
        "live_pairs_per_view": live_pv,
        "forward_ms_per_view": comp_ms.get("k_segsum", 0) + comp_ms.get("k_walk<kContrib>", 0),
        "backward_ms_per_view": comp_ms.get("k_replay<kGSum>", 0) + comp_ms.get("k_replay<kGrad>", 0),
        "live_pairs_per_s_fwd_bwd": live_pv / ((sum(comp_ms.values())) / 1e3) if sum(comp_ms.values()) else None,
        "ncu": {nm: ncu_traffic(nm)[2] for nm in COMPOSITING},
        "fp64_peak_tflops": 37.0, "fp64_peak_source": "B200 datasheet FP64 (vector) -- not measured here"}
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": L.KERNEL_NAMES[dom], "bytes_per_launch": bpl, "launch_ms": launch_ms,
                "launches_per_step": dom_per_step,
                "timing": "CUDA event nodes around each launch inside a single-stream graph of the step "
                          "(kernel alone on the GPU; last of the replays)",
                "share_of_instrumented_kernels": prof_ms[dom] / step_ms_all if step_ms_all else None,
                "kernel_ms_per_step": {L.KERNEL_NAMES[k]: round(prof_ms[k], 3) for k in L.KERNEL_NAMES},
                "per_view": {"t16": t16_pv, "live_pairs": live_pv, "items": items_pv},
                "traffic_source": traffic_src,
                "compute": dom_compute,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback 6.65 TB/s"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_label(args), "scene_order": args.scene_order,
                   "views_per_rank": V, "gaussians": args.n, "image": [args.size, args.size],
                   "param_dtype": args.param_dtype, "parallelism": f"view-sharded dp{world}",
                   "s_stop": step.s_stop, "l2": "inputs larger than L2 (112 MB params + ~0.3 GB/view records)",
                   "execution": f"one CUDA graph per step; K1-K5 batched per {step.geo_batch} views on a preprocessing stream, the views on {step.n_lanes} concurrent streams",
                   "t16_per_view": step.calib_t16_mean},
        "roofline": roofline,
        "stage_ms_per_step_single_stream": stages,
        "preprocess_sort_roofline": preprocess_sort_roofline(args.n, step, stages, V, peak),
        "compute_roofline": compute_roofline,
        "gpu_launches": int(launches),
        "e2e": e2e,
        "e2e_dropin": dropin,
        "clocks": clk.summary(),
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        procs = cpu_procs(args.cpu_procs)
        wall = cpu_run(host_scene, cfgs_all, procs, procs)
        line["cpu_baseline"] = {"value": procs / wall, "unit": UNIT, "cores": procs, "kind": "port",
                                "cpu": cpu_model(),
                                "sample": f"{procs} {args.workload} views ({args.n} Gaussians, {args.size}x{args.size}),"
                                          f" one per forked process, {wall:.1f} s wall"}
    if args.share_gpu:
        line["functional_check_only"] = (f"{world} ranks shared cuda:0 over {args.dist_backend}: exercises the "
                                         "multi-rank path, not a scaling measurement")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_sdgr(args)


if __name__ == "__main__":
    main()
