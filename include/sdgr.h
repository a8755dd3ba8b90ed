/*
 * sdgr.h — C ABI of the B200-native SAR Differentiable Gaussian Rasterizer.
 *
 * This is the drop-in boundary for the reference's hot path
 *   sarsplat.render / render_forward / backward
 * (/root/reference/pkg/src/sarsplat/forward.py:256-285, backward.py:243-290).
 * The reference is pure Python/NumPy, so its "FFI" for this path is the set of
 * stage functions its own tests call directly; each entry point below replaces
 * one of them (file:line cited per function).  INTEGRATION.md shows the ctypes
 * binding a maintainer of the reference would add.
 *
 * Conventions
 *  - Every pointer in the structs is a DEVICE pointer unless stated otherwise;
 *    all buffers are caller-allocated (the library never allocates).
 *  - Every call is asynchronous on the caller's `stream` (a cudaStream_t passed
 *    as void*; NULL = legacy default stream).  No call synchronises the host.
 *  - Return value: an sdgr_status code.  Device-side failures (a non-finite
 *    intensity, forward.py:192-196) are reported through the int32 status word
 *    the caller passes, read back once per step by the host wrapper.
 *  - Arrays indexed by Gaussian are N-sized in scene order (no compaction);
 *    culled / skipped Gaussians carry flags instead of being dropped.
 */
#ifndef SDGR_H_
#define SDGR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDGR_ABI_VERSION 2
#define SDGR_TILE 16          /* tile edge in cells / pixels (16x16 = 256 rays) */
#define SDGR_TILE_RAYS 256
#define SDGR_MAX_PLANE 32767  /* plane dims must fit int16 bboxes */
#ifndef SDGR_MAX_BATCH
#define SDGR_MAX_BATCH 24     /* views per batched call (*_batch); sdgr_max_batch() reports the build's */
#endif

typedef enum sdgr_status {
  SDGR_OK = 0,
  SDGR_ERR_INVALID = 1,   /* InvalidParameterError  (validation.py:16) */
  SDGR_ERR_NUMERICAL = 2, /* NumericalError         (validation.py:24) */
  SDGR_ERR_STATE = 3,     /* StateError             (validation.py:28) */
  SDGR_ERR_CUDA = 4,      /* a CUDA launch / runtime error               */
  SDGR_ERR_CAPACITY = 5   /* caller buffer too small (resize and retry)  */
} sdgr_status;

/* Gaussian flag bits (sdgr_projection.flags). */
#define SDGR_FLAG_VISIBLE 1u  /* passed skip + cull: Projection.indices (geometry.py:306) */
#define SDGR_FLAG_SKIPPED 2u  /* non-finite or det <= 0 (geometry.py:280-290)            */
#define SDGR_FLAG_CULLED 4u   /* outside the comp-plane 3-sigma frustum (geometry.py:293-305) */

/* Device status word layout (int32[4]) written by the compositing kernels. */
#define SDGR_STATUS_NONFINITE 0 /* != 0 when any per-pair contribution was non-finite */

/*
 * Per-view constants, filled on the host in FP64 with the reference's own
 * expressions (geometry.py:35-128) so they are bit-identical to it.
 */
typedef struct sdgr_view {
  double R[9];     /* world->radar rotation, row-major   (geometry.py:35-47)   */
  double T[3];     /* x_r = R x + T                       (geometry.py:59-62)   */
  double cam[3];   /* platform position                   (geometry.py:50-56)   */
  double mc[6];    /* jac_comp @ R, 2x3 row-major         (geometry.py:267)     */
  double mi[6];    /* jac_img  @ R                        (geometry.py:268)     */
  double den_u;    /* azimuth_res * n_azimuth             (geometry.py:85)      */
  double den_v;    /* range_res * n_range * tan(el)       (geometry.py:86,102)  */
  double off_vi;   /* 2 * altitude / (range_res*n_range*sin(el)) (geometry.py:103) */
  double cov_reg;  /* added to both 2D covariance diagonals (geometry.py:275-278) */
  double cutoff;   /* footprint radius; +inf = dense all-pairs mode (forward.py:80-84) */
  int32_t n_u, n_v;   /* computation-plane ray grid (radar.py:55-58) */
  int32_t n_az, n_rg; /* imaging-plane width (azimuth) / height (range) */
} sdgr_view;

/* Scene parameters, SoA like sarsplat.Scene (scene.py:132-158). */
typedef struct sdgr_scene {
  int64_t n;
  int32_t dtype;          /* 0 = float32, 1 = float64 */
  int32_t pad_;
  const void* positions;  /* (n,3) */
  const void* rotations;  /* (n,4) w,x,y,z (need not be unit) */
  const void* log_scales; /* (n,3) */
  const void* sh_coeffs;  /* (n,16) */
  const void* ke_raw;     /* (n,2) softplus pre-activations */
} sdgr_scene;

/* One projection plane's footprint records (N-sized).  With both `packed` and
 * `emit` given (multi-view steps), uv, bbox, cell_mask and tile_mask may be
 * NULL: sdgr_project then skips them and the binning reads the rows. */
typedef struct sdgr_plane {
  double* uv;           /* (n,2) pixel-space center                          */
  double* inv_cov;      /* (n,4) a00, a01, a11, 0  (forward.py:33-42)        */
  double* cov;          /* (n,4) c00, c01, c11, 0  optional (NULL = skip)     */
  int16_t* bbox;        /* (n,4) x0, x1, y0, y1 clipped cell bbox (forward.py:76-79) */
  uint64_t* cell_mask;  /* (n) members in the 8x8 cell window at (x0,y0), bit = (iv-y0)*8+(iu-x0) */
  uint64_t* tile_mask;  /* (n) member tiles in the 8x8 tile window at (x0/16,y0/16) */
  int32_t* n_tiles;     /* (n) number of 16x16 tiles holding >= 1 member cell */
  double* packed;       /* (n,8) optional, computation plane only (NULL = skip): per visible
                           Gaussian u, v, a00, a01, a11, kappa, phase, cell_mask (bits) in one
                           64-byte row, so the pair-record gather reads 2 sectors, not 6 */
  uint64_t* emit;       /* (n,2) optional (NULL = skip): bbox (4 x int16) and tile_mask in one
                           16-byte row per Gaussian, for the fused count + emit pass of
                           sdgr_bin_batch (1 random sector per Gaussian instead of 4) */
} sdgr_plane;

/* Output of sdgr_project (geometry.Projection, geometry.py:185-230). */
typedef struct sdgr_projection {
  int64_t n;
  sdgr_plane comp;       /* computation plane (n_u x n_v)   */
  sdgr_plane img;        /* imaging plane (n_az x n_rg)     */
  uint64_t* depth_key;   /* (n) order-preserving FP64 depth key; UINT64_MAX if not visible;
                            16-byte aligned (sdgr_depth_order* read it in 16-byte loads) */
  double* kappa;         /* (n) ke_fwd + ke_bwd (geometry.py:317, Projection.ke_sum); NULL if comp.packed */
  double* phase;         /* (n) max(0, P~)                  (geometry.py:316); NULL if comp.packed */
  double* phase_raw;     /* (n) P~ (backward clamp gate)    (geometry.py:315) */
  uint8_t* flags;        /* (n) SDGR_FLAG_* */
  int32_t* counters;     /* (4) [0] visible, [1] skipped, [2] culled; zeroed by sdgr_project */
  /* optional accessors (NULL to skip) */
  double* ke_act;        /* (n,2) softplus(ke_raw)          */
  double* look;          /* (n,4) unit look dir xyz, distance (geometry.py:308-313) */
  unsigned long long* member_pairs; /* (2) member (cell, Gaussian) pairs T_c, T_i; optional */
} sdgr_projection;

/* Live-pair replay log, written by sdgr_composite_forward and consumed by
 * sdgr_grad_intensity: for every live (ray, Gaussian) pair of the computation
 * plane -- in each ray's walk order -- the log-transmittance before the pair
 * and its footprint weight, grouped by walk sub-chunk.  The backward then
 * touches only live pairs (no re-binning, no membership, no weights). */
typedef struct sdgr_replay {
  int64_t capacity;      /* pair slots; T_c (member_pairs[0]) always suffices */
  double* y1;            /* (capacity) T (1 - e^-tau): transmittance x opacity */
  double* t2;            /* (capacity) T e^-tau: transmittance after the pair  */
  double* w;             /* (capacity) footprint weight exp(-q)            */
  uint8_t* j;            /* (capacity) Gaussian index within its chunk      */
  uint8_t* r;            /* (capacity) ray index within its tile            */
  int32_t desc_per_item; /* descriptor slots per work item                  */
  int32_t pad_;
  int32_t* desc;         /* (max_items*desc_per_item, 4): offset, count, chunk start, j0 | j1 << 16 */
  int32_t* desc_count;   /* (max_items) descriptors written per item        */
  unsigned long long* cursor; /* (2) device cursor [0], zeroed by the forward, and a
                                 sticky overflow flag [1] the caller zeroes */
  double* gpair;         /* (tiles->n_pairs) scratch: dL/dI per sorted pair, written by
                            the first backward replay pass, read by the second */
} sdgr_replay;

/* Packed per-(tile, Gaussian) record, one per sorted pair of the computation
 * plane, so the ordered tile walks read their inputs coalesced (80 B). */
typedef struct sdgr_pair_rec {
  double u, v;              /* computation-plane center              */
  double a00, a01, a11;     /* inverse covariance                    */
  double kappa, phase;      /* ke_fwd + ke_bwd, max(0, P~)           */
  uint64_t cell_mask;       /* 8x8 member window at (bbox.x0, bbox.y0) */
  int16_t x0, x1, y0, y1;   /* clipped cell bbox                      */
  int32_t pos;              /* pre-sort position (partial-record index) */
  int32_t prim;             /* scene index                           */
} sdgr_pair_rec;

/* (tile, Gaussian) binning of one plane: the per-tile key lists.
 * Pairs are emitted per Gaussian in list order (rank order on the computation
 * plane, index order on the imaging plane) at "pre-sort positions"; Gaussian g
 * owns the contiguous pre-sort range [pair_start[g], pair_start[g]+n_tiles[g]).
 * Per-pair partial sums are stored by pre-sort position so the per-Gaussian
 * reductions run in a fixed order (deterministic, atomic-free). */
typedef struct sdgr_tiles {
  int32_t plane;        /* 0 = computation (depth order), 1 = imaging (index order) */
  int32_t tiles_x, tiles_y, n_tiles;
  int64_t n_pairs;      /* T16: number of (tile, Gaussian) member pairs */
  uint32_t* pair_tile;  /* (n_pairs) tile id, sorted ascending              */
  int32_t* pair_pos;    /* (n_pairs) pre-sort position of each sorted pair    */
  int32_t* pair_prim;   /* (n_pairs) scene index; per tile by (depth, index) or index */
  int32_t* pre_prim;    /* (n_pairs) scene index by pre-sort position         */
  int32_t* pair_start;  /* (n) first pre-sort position of each Gaussian       */
  int32_t* tile_range;  /* (n_tiles,2) [start, end) into the sorted arrays    */
  int32_t seg_len;      /* max Gaussians per work item (depth segment)       */
  int32_t max_items;    /* capacity of items                                  */
  int32_t device_count; /* 1: n_pairs is a capacity; the exact count stays on the
                           device (offsets[n]) so no host round trip is needed */
  int32_t pad_;
  int32_t* items;       /* (max_items,4) tile, start, end; column 3 = the
                           processing order (row c: the item the c-th
                           claim of a persistent walk takes)             */
  int32_t* tile_first;  /* (n_tiles) index of each tile's first work item     */
  int32_t* n_items;     /* (4) device: [0] work items, [1] overflow flag, [2] walk counter */
  sdgr_pair_rec* pair_rec; /* (n_pairs) packed per-pair records in sorted order
                              (computation plane; filled by sdgr_bin_pairs)   */
} sdgr_tiles;

/* Scene gradients (backward.SceneGradients, backward.py:25-50).
 * dtype selects the element type of every gradient array: 0 = float32
 * (device training steps), 1 = float64 (host callers: the reference returns
 * FP64).  visible_dtype: 0 = int32 view counts, 1 = counts stored in `dtype`
 * (exact below 2^24 in float32), so a flat multi-view gradient buffer is
 * summed across ranks by ONE all-reduce. */
typedef struct sdgr_grads {
  int32_t dtype;
  int32_t visible_dtype;
  void* positions;      /* (n,3)  */
  void* rotations;      /* (n,4)  */
  void* log_scales;     /* (n,3)  */
  void* sh_coeffs;      /* (n,16) */
  void* ke_raw;         /* (n,2)  */
  void* uv_grad_norm;   /* (n)    */
  void* visible;        /* (n) 1 if visible (accumulate mode: count of views) */
} sdgr_grads;

/* ---------------------------------------------------------------- misc -- */
int sdgr_version(void);
const char* sdgr_status_string(int status);
/* Kernels launched by this library since load (the bench's gpu_launches). */
uint64_t sdgr_launch_count(void);
/* SDGR_MAX_BATCH of this build (views per *_batch call). */
int sdgr_max_batch(void);
/* Device timing of selected kernels: between sdgr_profile_begin(mask) and
 * sdgr_profile_end, every launch of a kernel whose bit (1 << SDGR_K_*) is in
 * mask is bracketed by CUDA events on its launch stream.  sdgr_profile_end
 * synchronises on the last event and returns per-kernel totals (ms) and
 * launch counts in arrays of SDGR_PROFILE_KERNELS entries (index = SDGR_K_*).
 * Used by bench.py to time the dominant kernel inside the timed region. */
#define SDGR_PROFILE_KERNELS 16
#define SDGR_K_PROJECT 1      /* K1 k_project                      */
#define SDGR_K_ONESWEEP 2     /* radix sort passes (depth + tile)  */
#define SDGR_K_EMIT 3         /* pair emission (fused count + emit in batches) */
#define SDGR_K_GATHER 4       /* pair record packing               */
#define SDGR_K_SEGSUM 5       /* forward pass A (segment sums)     */
#define SDGR_K_WALK 6         /* forward tile walk (contributions) */
#define SDGR_K_SPLAT 7        /* imaging-plane splat               */
#define SDGR_K_GRAD_IMAGE 8   /* imaging-plane backward            */
#define SDGR_K_REPLAY_GSUM 9  /* backward replay, segment sums     */
#define SDGR_K_REPLAY_GRAD 10 /* backward replay, gradients        */
#define SDGR_K_GEOMETRY 11    /* per-Gaussian chain rule (batched) */
int sdgr_profile_begin(uint32_t kernel_mask);
int sdgr_profile_end(double* ms, int64_t* launches);
/* Before sdgr_profile_end: the recorded launches as a timeline -- kernel id
 * (SDGR_K_*) and the begin / end event times (ms) relative to the first
 * recorded begin, up to cap entries; returns the count (negative status on
 * error).  Events are stream-ordered markers: begin fires when the launch
 * stream reaches the kernel, so with concurrent streams [begin, end] is the
 * span from "ready" to "done". */
int sdgr_profile_timeline(int cap, int32_t* ids, double* t0_ms, double* t1_ms);
/* Page-lock a caller's host buffer for direct DMA (cudaHostRegister,
 * portable) / release it.  The drop-in host path registers scene arrays it
 * sees again on a later call (the reference's training loop updates them in
 * place, optimize.py:206) so their uploads skip the staging copy.  Returns
 * SDGR_OK or -SDGR_ERR_CUDA (e.g. the pages overlap another registration);
 * a failure never leaves a pending CUDA error behind. */
int sdgr_host_register(void* ptr, size_t bytes);
int sdgr_host_unregister(void* ptr);
/* Bytes of scratch the binning calls need for n Gaussians / max pairs. */
size_t sdgr_workspace_bytes(int64_t n, int64_t max_pairs);
/* ... and the batched calls for n_views (1..SDGR_MAX_BATCH) views (0 if n_views is out of range). */
size_t sdgr_batch_workspace_bytes(int64_t n, int64_t max_pairs, int n_views);

/* ------------------------------------------------ preprocess (K1) -------- */
/* geometry.project_all (geometry.py:233-340) + the footprint bbox / member
 * tests of forward._footprint_pairs (forward.py:60-109) for both planes. */
int sdgr_project(const sdgr_scene* scene, const sdgr_view* view,
                 sdgr_projection* proj, void* stream);
/* sdgr_project for n_views (1..SDGR_MAX_BATCH) views of one scene in one
 * launch: views[k] -> projs[k], each exactly as the single-view call.  The
 * parameters are read once and their view-independent half (normalised
 * quaternion, R(q), e^s, Sigma = M M^T, softplus extinctions) is computed once
 * per Gaussian for the whole batch (a multi-view step's preprocessing). */
int sdgr_project_batch(const sdgr_scene* scene, int n_views, const sdgr_view* views,
                       sdgr_projection* projs, void* stream);

/* --------------------------------------------------- binning (K2-K5) ----- */
/* Stable sort of the visible Gaussians by (depth, index): order[rank] = g.
 * The depth half of np.lexsort((prim, depth, cell)) (forward.py:147). */
int sdgr_depth_order(const sdgr_projection* proj, int32_t* order,
                     void* ws, size_t ws_bytes, void* stream);
/* sdgr_depth_order for n_views projections of one scene (orders[k] <- projs[k]),
 * every radix pass one launch over all views.  ws: sdgr_batch_workspace_bytes. */
int sdgr_depth_order_batch(int n_views, const sdgr_projection* projs, int32_t* const* orders,
                           void* ws, size_t ws_bytes, void* stream);
/* offsets[i] = exclusive prefix of member-tile counts in rank order (plane 0,
 * `order` given) or scene order (plane 1, order == NULL); offsets has n+1
 * entries, offsets[n] = T16 for the plane. */
int sdgr_count_pairs(const sdgr_projection* proj, int32_t plane,
                     const int32_t* order, int32_t* offsets,
                     void* ws, size_t ws_bytes, void* stream);
/* Emit (tile, Gaussian) pairs, stable-sort them by tile, extract tile
 * ranges and depth-segment work items: the per-tile key lists
 * (forward.py:138-155 at 16x16 granularity; _build_splat_pairs :213-224). */
int sdgr_bin_pairs(const sdgr_projection* proj, const sdgr_view* view,
                   const int32_t* order, const int32_t* offsets,
                   sdgr_tiles* tiles, void* ws, size_t ws_bytes, void* stream);
/* sdgr_count_pairs + sdgr_bin_pairs of one plane for n_views views, each
 * stage one launch over all views: orders[k] (plane 0) / NULL (plane 1),
 * offsets[k] (n+1, written), tiles[k] (same tile grid, capacity and
 * device_count for every view).  ws: sdgr_batch_workspace_bytes. */
int sdgr_bin_batch(int n_views, const sdgr_projection* projs, const sdgr_view* views, int32_t plane,
                   const int32_t* const* orders, int32_t* const* offsets, sdgr_tiles* tiles,
                   void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------- forward (K6, K7) ------ */
/* compute_intensities (forward.py:178-199): per-ray emission-absorption walk.
 * seg_sum / seg_base: (max_items*256) FP64 per-(item, ray) optical-depth
 * segment sums and exclusive prefixes (kept for the backward).
 * partial_I: (n_pairs) FP64 per-(tile, Gaussian) partial intensities.
 * intensity: (n) FP64, overwritten.  s_stop: rays stop once their
 * log-transmittance exceeds it (+inf = never, the reference's behaviour).
 * status: int32[4]; [0] != 0 if any contribution was non-finite.
 * replay: optional (NULL = none) live-pair log for sdgr_grad_intensity. */
int sdgr_composite_forward(const sdgr_view* view, const sdgr_projection* proj,
                           const sdgr_tiles* comp, double s_stop,
                           double* seg_sum, double* seg_base, double* partial_I,
                           double* intensity, int32_t* status, sdgr_replay* replay,
                           void* stream);
/* splat_image (forward.py:227-240): image (n_rg, n_az) FP64 overwritten.
 * Gaussian-parallel with deterministic fixed-point accumulation (u64 sums of
 * w I * 2^(47-e), 2^e > the view's largest intensity: absolute precision
 * 2^-47 of the brightest Gaussian, bitwise reproducible), so it needs no
 * imaging-plane lists.  scratch: (n_rg*n_az + 1) * 8 bytes. */
int sdgr_splat(const sdgr_view* view, const sdgr_projection* proj,
               const double* intensity, void* scratch, double* image, void* stream);

/* ------------------------------------------------ backward (K8-K10) ------ */
/* grad_image_stage (backward.py:86-104).  dL_dS: (n_rg, n_az) FP64.
 * acc_img (6,n) FP64: dL/dI, dL/dA(3), dL/duv(2) on the imaging plane
 * (A = inverse covariance). */
int sdgr_grad_image(const sdgr_view* view, const sdgr_projection* proj,
                    const double* intensity, const double* dL_dS, double* acc_img,
                    void* stream);
/* grad_intensity_stage (backward.py:107-148).  dL_dI = acc_img row 0.
 * partial_g: (n_pairs, 8) FP64 per-(tile, Gaussian) partials of dL/dP,
 * dL/dkappa, dL/dA(3), dL/duv(2) on the computation plane.
 * seg_g / seg_d: (max_items*256) FP64 scratch.
 * replay: the log the forward wrote (NULL = re-walk the tile lists). */
int sdgr_grad_intensity(const sdgr_view* view, const sdgr_projection* proj,
                        const sdgr_tiles* comp, double s_stop,
                        const double* seg_base, const double* dL_dI,
                        double* seg_g, double* seg_d, double* partial_g,
                        const sdgr_replay* replay, void* stream);
/* grad_geometry_stage + grad_sh_stage + the final scatter (backward.py:171-290).
 * Reduces partial_g per Gaussian (fixed order) and chains to parameters.
 * accumulate = 0 overwrites `out`, 1 adds into it (multi-view steps). */
int sdgr_grad_geometry(const sdgr_scene* scene, const sdgr_view* view,
                       const sdgr_projection* proj, const sdgr_tiles* comp,
                       const double* acc_img, const double* partial_g,
                       sdgr_grads* out, int accumulate, void* stream);
/* sdgr_grad_geometry over n_views (1..SDGR_MAX_BATCH) views of one scene in
 * one pass: arrays of length n_views, element k describing view k exactly as
 * the single-view call does.  The per-view terms are summed in FP64 before
 * the (linear) covariance chain and the single read-modify-write of `out`,
 * so a batch equals the sum of its views up to rounding.  Multi-view steps
 * (optimize.py:395-425 accumulation) use it to pay the scene loads and the
 * gradient update once per batch. */
int sdgr_grad_geometry_batch(const sdgr_scene* scene, int n_views, const sdgr_view* views,
                             const sdgr_projection* projs, const sdgr_tiles* comps,
                             const double* const* acc_imgs, const double* const* partial_gs,
                             sdgr_grads* out, int accumulate, void* stream);

/* ------------------------ reference-shaped stage outputs (accessors) ---- */
/* The fused path above keeps per-Gaussian and per-(tile, Gaussian) state.
 * These calls expose what the reference's stage functions return, for
 * callers and tests that use the stage API (tests/test_forward.py,
 * tests/test_backward.py drive those functions directly). */
/* forward._footprint_pairs + build_ray_lists / _build_splat_pairs
 * (forward.py:60-155, 213-224): the member (cell, Gaussian) pairs of one
 * plane in the reference's order -- cell-major, then (depth, index) on the
 * computation plane, index on the imaging plane -- from the plane's tile
 * lists.  Needs the projection's SoA records (uv, inv_cov, bbox, cell_mask).
 * Call 1 (prim == NULL): offsets (n_cells + 1, int64) <- CSR of the member
 * counts per cell (n_cells = n_u*n_v or n_az*n_rg, cell = iv*width + iu).
 * Call 2: prim (scene index), delta (dx, dy), q and w = exp(-q) of the
 * offsets[n_cells] pairs. */
int sdgr_cell_pairs(const sdgr_projection* proj, const sdgr_view* view, const sdgr_tiles* tiles,
                    int64_t* offsets, int32_t* prim, double* delta, double* q, double* w, void* stream);
/* compute_intensities' per-pair buffers (forward.py:167-199) over the
 * computation-plane pairs of sdgr_cell_pairs: tau, trans, absorb, contrib
 * (each ray's exclusive log-transmittance prefix in list order).  Needs
 * proj->kappa and proj->phase. */
/* Diagnostics: y[i] = the compositing path's e^x (nexp, common.cuh) for n
 * device doubles -- its accuracy against libdevice exp is tested. */
int sdgr_exp_check(int64_t n, const double* x, double* y, void* stream);
int sdgr_cell_intensities(const sdgr_projection* proj, int64_t n_cells, const int64_t* offsets,
                          const int32_t* prim, const double* w, double* tau, double* trans,
                          double* absorb, double* contrib, void* stream);
/* grad_image_stage's per-pair dL/dbeta = dL/dS[pixel] * I[prim] (backward.py:99). */
int sdgr_splat_pair_grads(int64_t n_pairs, const int32_t* pair_pixel, const int32_t* pair_prim,
                          const double* dL_dS, const double* intensity, double* dL_dbeta, void* stream);
/* Per-Gaussian plane-space gradients, (8, n) FP64 rows:
 * plane 0 from sdgr_grad_intensity's partial_g: dL/dP, dL/dkappa,
 *   dL/dSigma_c (2x2 row-major), dL/du, dL/dv (grad_intensity_stage, backward.py:107-148);
 * plane 1 from sdgr_grad_image's acc_img: dL/dI, 0, dL/dSigma_i, dL/du, dL/dv
 *   (grad_image_stage, backward.py:86-104).  comp: the plane-0 tiles (NULL for plane 1). */
int sdgr_stage_grads(const sdgr_projection* proj, int32_t plane, const sdgr_tiles* comp,
                     const double* src, double* out, void* stream);
/* grad_geometry_stage + grad_sh_stage + the scatter (backward.py:171-290)
 * from caller-given plane-space gradients ex (14, n) FP64 rows:
 * dSigma_c (4), dSigma_i (4), duv_c (2), duv_i (2), dP, dkappa.  out overwritten. */
int sdgr_grad_geometry_explicit(const sdgr_scene* scene, const sdgr_view* view, const sdgr_projection* proj,
                                const double* ex, sdgr_grads* out, void* stream);
/* A projection given in plane space (the reference tests' hand-assembled
 * Projection, tests/test_forward.py:43-59): n rows, all visible; per plane
 * uv (n,2) and covariance (n,3: c00, c01, c11), depth (n), phase_raw (n,
 * P before the clamp), kappa (n) -> the records sdgr_project would write for
 * the same plane-space values (footprints, depth keys, packed rows). */
int sdgr_project_planes(const sdgr_view* view, int64_t n, const double* uv_comp, const double* uv_img,
                        const double* depth, const double* cov_comp, const double* cov_img,
                        const double* phase_raw, const double* kappa, sdgr_projection* proj, void* stream);

/* ----------------------------------- training step -- */
/* optimize.loss (optimize.py:85-102): value = (1-l) mean|S-Y| + l (1 - SSIM(S,Y))
 * and dL_dS (h, w) FP64, SSIM with its analytic gradient (metrics.py:98-137):
 * 11x11 separable Gaussian window (sigma 1.5, `kernel11` = its 11 normalised
 * taps in HOST memory, zero padded), interior mean; images smaller than the
 * window use one global window.  value: device FP64 scalar.  scratch:
 * sdgr_loss_scratch_bytes(h, w).  lambda_ssim in [0, 1]. */
size_t sdgr_loss_scratch_bytes(int h, int w);
int sdgr_loss(const double* S, const double* Y, int h, int w, double lambda_ssim, double max_val,
              const double* kernel11, double* value, double* dL_dS, void* scratch, void* stream);
/* optimize.adam_step (optimize.py:171-207), in place on `scene`; `m` and `v`
 * are scenes of the same dtype/shape holding the moment buffers; grads are the
 * FP32 SceneGradients.  lr[5] per group (positions, rotations, log_scales,
 * sh_coeffs, ke_raw); bc1 = 1 - beta1^step, bc2 = 1 - beta2^step computed by
 * the caller; displacement_bound <= 0 disables the clamp.  Non-finite
 * gradient entries are zeroed and added to *n_skipped (device u64).  grads
 * must be float32 (dtype 0).  guard: optional device int32; when it is
 * non-zero at run time the whole update is skipped (a multi-view step whose
 * pair buffers overflowed produced truncated gradients -- MultiViewStep's
 * overflow word -- so the step can be recalibrated and re-run exactly). */
int sdgr_adam_step(sdgr_scene* scene, const sdgr_grads* grads, sdgr_scene* m, sdgr_scene* v,
                   const double* lr, double beta1, double beta2, double eps, double bc1, double bc2,
                   double displacement_bound, unsigned long long* n_skipped, const int32_t* guard,
                   void* stream);

/* -------------------------------- densification ------ */
/* optimize.densify_and_prune (optimize.py:251-312) and GradAccumulator
 * (:217-239) as device passes; the caller gathers rows with the index lists
 * the flags define, and draws the split samples xi from its own seeded
 * generator (rng.normal(size=(2 * n_split, 3)), as the reference does). */
/* norm_sum += uv_grad_norm, pos_sum (n,3) += positions, count += visible for
 * rows with visible > 0 (visible = views that saw the Gaussian). FP64 sums;
 * grads float32 (dtype 0), visible int32 or float32 counts. */
int sdgr_accum_update(const sdgr_grads* grads, int64_t n, double* norm_sum, double* pos_sum,
                      double* count, void* stream);
/* flags[g] = 2 split (max e^s > cap), 1 clone (mean norm > grad_thr, small,
 * seen), 0 keep.  small: max e^s <= small_size. */
int sdgr_densify_flags(const sdgr_scene* scene, const double* norm_sum, const double* count, double cap,
                       double small_size, double grad_thr, uint8_t* flags, void* stream);
/* in place on gathered clone rows: positions += -position_lr * pos_sum / max(count, 1) */
int sdgr_clone_shift(sdgr_scene* clones, const double* pos_sum, const double* count, double position_lr,
                     void* stream);
/* in place on gathered child rows (each parent twice): positions += chol(Sigma) xi (xi: (n,3) FP64),
 * log_scales -= log_shrink */
int sdgr_split_children(sdgr_scene* children, const double* xi, double log_shrink, void* stream);
/* survive[g] = DC phase (sh_0 * SH_C0) >= phase_floor and max e^s <= cap */
int sdgr_prune_flags(const sdgr_scene* scene, double cap, double phase_floor, uint8_t* survive, void* stream);

/* ---------------------------- scene checkpoints ---- */
/* The reference's binary PLY vertex records (ply.py:110-155): per Gaussian 28
 * little-endian doubles, x y z qw qx qy qz log_scale_xyz sh_0..15 ke_fwd ke_bwd.
 * pack: scene (f32/f64 SoA) -> out (n * 28 doubles, vertex-major).
 * unpack: in (n vertices of `stride` doubles) -> scene; col[k] (host, 28
 * ints) = column of scene property k in a vertex. */
int sdgr_ply_pack(const sdgr_scene* scene, double* out, void* stream);
int sdgr_ply_unpack(const double* in, int64_t n, int stride, const int32_t* col, sdgr_scene* scene,
                    void* stream);

/* ------------------------------ point-cloud evaluation -- */
/* metrics.chamfer / precision_recall_f1 / dbscan_inlier_mask (metrics.py:140-183)
 * on a uniform grid of dims[0] x dims[1] x dims[2] cells (<= 2^24) of edge h
 * with corner lo (host arrays).  Points are (n,3) FP64 device arrays.
 * ws: sdgr_grid_workspace_bytes(n of the gridded set, cells). */
size_t sdgr_grid_workspace_bytes(int64_t n, int64_t n_cells);
/* d2[i] = squared distance from query i to its nearest reference point (the
 * cKDTree query of metrics.py:150-151, 159-160), exact, FP64. */
int sdgr_nn_sqdist(const double* ref, int64_t n_ref, const double* query, int64_t n_query,
                   const double* lo, double h, const int32_t* dims, double* d2,
                   void* ws, size_t ws_bytes, void* stream);
/* DBSCAN (sklearn semantics, metrics.py:165-177): root[i] = the smallest core
 * index of point i's cluster (core: >= min_pts points within eps, itself
 * included; border points join the cluster the reference's index-order
 * expansion reaches first), -1 for noise.  Requires h >= eps. */
int sdgr_dbscan(const double* pts, int64_t n, const double* lo, double h, const int32_t* dims,
                double eps, int32_t min_pts, int32_t* root, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SDGR_H_ */
