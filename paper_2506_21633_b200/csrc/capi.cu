// capi.cu — extern "C" entry points of libsdgr (include/sdgr.h).
//
// Thin argument checking + dispatch to the stream-ordered launchers.  No
// host synchronisation, no allocation, no C++ exceptions across the ABI.
#include <atomic>
#include <cmath>

#include "common.cuh"

namespace sdgr {

static std::atomic<uint64_t> g_launches{0};
void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
int check_launch() { return cudaPeekAtLastError() == cudaSuccess ? SDGR_OK : SDGR_ERR_CUDA; }

// ---- kernel timing: a pool of event pairs recorded around selected launches
constexpr int kProfMax = 16384;
static uint32_t g_prof_mask = 0;
static cudaEvent_t g_prof_ev[2 * kProfMax];
static int g_prof_id[kProfMax];
static int g_prof_created = 0, g_prof_n = 0;
static bool g_prof_open = false;

// inside a stream capture the records must be external event nodes (a
// default-flag record only orders the capture and never fires on replay)
static void prof_record(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  else
    cudaEventRecord(ev, st);
}

void prof_mark(int id, bool begin, cudaStream_t st) {
  if (!(g_prof_mask & (1u << id))) return;
  if (begin) {
    if (g_prof_n >= kProfMax) return;
    if (g_prof_n >= g_prof_created) {
      cudaEventCreate(&g_prof_ev[2 * g_prof_n]);
      cudaEventCreate(&g_prof_ev[2 * g_prof_n + 1]);
      g_prof_created = g_prof_n + 1;
    }
    prof_record(g_prof_ev[2 * g_prof_n], st);
    g_prof_id[g_prof_n] = id;
    g_prof_open = true;
  } else if (g_prof_open) {
    prof_record(g_prof_ev[2 * g_prof_n + 1], st);
    ++g_prof_n;
    g_prof_open = false;
  }
}

int launch_project(const sdgr_scene&, int, const sdgr_view*, sdgr_projection*, cudaStream_t);
int launch_depth_order_batch(int, const sdgr_projection*, int32_t* const*, void*, size_t, cudaStream_t);
int launch_count_batch(int, const int32_t* const*, const int32_t* const*, int64_t, int32_t* const*, void*, size_t,
                       cudaStream_t);
int launch_bin_batch(int, const sdgr_projection*, const sdgr_view*, int, const int32_t* const*, int32_t* const*,
                     sdgr_tiles*, bool, void*, size_t, cudaStream_t);
size_t batch_ws_bytes(int64_t, int64_t, int);
int launch_composite_forward(const sdgr_view&, const sdgr_projection&, const sdgr_tiles&, double,
                             double*, double*, double*, double*, int32_t*, const sdgr_replay*, cudaStream_t);
int launch_splat(const sdgr_view&, const sdgr_projection&, const double*, double*, double*,
                 cudaStream_t);
int launch_grad_image(const sdgr_view&, const sdgr_projection&, const double*, const double*, double*,
                      cudaStream_t);
int launch_grad_intensity(const sdgr_view&, const sdgr_projection&, const sdgr_tiles&, double,
                          const double*, const double*, double*, double*, double*, const sdgr_replay*,
                          cudaStream_t);

size_t loss_scratch_bytes(int, int);
int launch_loss(const double*, const double*, int, int, double, double, const double*, double*, double*, void*,
                cudaStream_t);
int launch_adam(const sdgr_scene&, const sdgr_grads&, const sdgr_scene&, const sdgr_scene&, const double*, double,
                double, double, double, double, double, unsigned long long*, const int32_t*, cudaStream_t);

int launch_accum_update(const sdgr_grads&, int64_t, double*, double*, double*, cudaStream_t);
int launch_cell_pairs(const sdgr_projection&, const sdgr_view&, const sdgr_tiles&, int64_t*, int32_t*, double*,
                      double*, double*, cudaStream_t);
int launch_exp_check(int64_t, const double*, double*, cudaStream_t);
int launch_cell_intensities(const sdgr_projection&, int64_t, const int64_t*, const int32_t*, const double*, double*,
                            double*, double*, double*, cudaStream_t);
int launch_splat_pair_grads(int64_t, const int32_t*, const int32_t*, const double*, const double*, double*,
                            cudaStream_t);
int launch_stage_grads(const sdgr_projection&, int, const sdgr_tiles*, const double*, double*, cudaStream_t);
int launch_grad_geometry_explicit(const sdgr_scene&, const sdgr_view&, const sdgr_projection&, const double*,
                                  const sdgr_grads&, cudaStream_t);
int launch_project_planes(const sdgr_view&, int64_t, const double*, const double*, const double*, const double*,
                          const double*, const double*, const double*, const sdgr_projection&, cudaStream_t);
int launch_densify_flags(const sdgr_scene&, const double*, const double*, double, double, double, uint8_t*,
                         cudaStream_t);
int launch_clone_shift(const sdgr_scene&, const double*, const double*, double, cudaStream_t);
int launch_split_children(const sdgr_scene&, const double*, double, cudaStream_t);
int launch_prune_flags(const sdgr_scene&, double, double, double, uint8_t*, cudaStream_t);

int launch_ply_pack(const sdgr_scene&, double*, cudaStream_t);
int launch_ply_unpack(const double*, int64_t, int, const int32_t*, const sdgr_scene&, cudaStream_t);

static bool replay_ok(const sdgr_replay* r) {
  return !r || (r->y1 && r->t2 && r->w && r->j && r->r && r->desc && r->desc_count && r->cursor && r->gpair && r->capacity > 0 &&
                r->desc_per_item > 0);
}
int launch_grad_geometry(const sdgr_scene&, int, const sdgr_view*, const sdgr_projection*, const sdgr_tiles*,
                         const double* const*, const double* const*, const sdgr_grads&, int, cudaStream_t);

static bool view_ok(const sdgr_view* v) {
  if (!v) return false;
  if (v->n_u < 1 || v->n_v < 1 || v->n_az < 1 || v->n_rg < 1) return false;
  if (v->n_u > SDGR_MAX_PLANE || v->n_v > SDGR_MAX_PLANE || v->n_az > SDGR_MAX_PLANE ||
      v->n_rg > SDGR_MAX_PLANE)
    return false;
  if (std::isnan(v->cutoff) || v->cutoff < 0) return false;
  return true;
}

static bool tiles_ok(const sdgr_tiles* t) {
  return t && t->n_tiles >= 1 && t->tiles_x >= 1 && t->seg_len >= 1 && t->max_items >= 1 &&
         t->tile_range && t->items && t->tile_first && t->n_items;
}

}  // namespace sdgr

using namespace sdgr;

extern "C" {

int sdgr_version(void) { return SDGR_ABI_VERSION; }

const char* sdgr_status_string(int s) {
  switch (s) {
    case SDGR_OK: return "ok";
    case SDGR_ERR_INVALID: return "invalid parameter";
    case SDGR_ERR_NUMERICAL: return "non-finite value";
    case SDGR_ERR_STATE: return "invalid state";
    case SDGR_ERR_CUDA: return cudaGetErrorString(cudaGetLastError());
    case SDGR_ERR_CAPACITY: return "buffer capacity exceeded";
    default: return "unknown status";
  }
}

uint64_t sdgr_launch_count(void) { return g_launches.load(); }

int sdgr_max_batch(void) { return SDGR_MAX_BATCH; }

int sdgr_profile_begin(uint32_t kernel_mask) {
  g_prof_mask = kernel_mask;
  g_prof_n = 0;
  g_prof_open = false;
  return SDGR_OK;
}

int sdgr_profile_end(double* ms, int64_t* launches) {
  g_prof_mask = 0;
  if (!ms || !launches) return SDGR_ERR_INVALID;
  for (int k = 0; k < SDGR_PROFILE_KERNELS; ++k) { ms[k] = 0.0; launches[k] = 0; }
  if (g_prof_n > 0 && cudaEventSynchronize(g_prof_ev[2 * g_prof_n - 1]) != cudaSuccess) return SDGR_ERR_CUDA;
  for (int i = 0; i < g_prof_n; ++i) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, g_prof_ev[2 * i], g_prof_ev[2 * i + 1]) != cudaSuccess) return SDGR_ERR_CUDA;
    ms[g_prof_id[i]] += t;
    launches[g_prof_id[i]] += 1;
  }
  g_prof_n = 0;
  return SDGR_OK;
}

int sdgr_profile_timeline(int cap, int32_t* ids, double* t0_ms, double* t1_ms) {
  if (cap < 0 || (cap > 0 && (!ids || !t0_ms || !t1_ms))) return -SDGR_ERR_INVALID;
  if (g_prof_n == 0) return 0;
  if (cudaEventSynchronize(g_prof_ev[2 * g_prof_n - 1]) != cudaSuccess) return -SDGR_ERR_CUDA;
  const int n = g_prof_n < cap ? g_prof_n : cap;
  for (int i = 0; i < n; ++i) {
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, g_prof_ev[0], g_prof_ev[2 * i]) != cudaSuccess ||
        cudaEventElapsedTime(&b, g_prof_ev[0], g_prof_ev[2 * i + 1]) != cudaSuccess)
      return -SDGR_ERR_CUDA;
    ids[i] = g_prof_id[i];
    t0_ms[i] = a;
    t1_ms[i] = b;
  }
  return n;
}

int sdgr_host_register(void* ptr, size_t bytes) {
  if (!ptr || bytes == 0) return -SDGR_ERR_INVALID;
  if (cudaHostRegister(ptr, bytes, cudaHostRegisterPortable) != cudaSuccess) {
    (void)cudaGetLastError();
    return -SDGR_ERR_CUDA;
  }
  return SDGR_OK;
}

int sdgr_host_unregister(void* ptr) {
  if (!ptr) return -SDGR_ERR_INVALID;
  if (cudaHostUnregister(ptr) != cudaSuccess) {
    (void)cudaGetLastError();
    return -SDGR_ERR_CUDA;
  }
  return SDGR_OK;
}

size_t sdgr_workspace_bytes(int64_t n, int64_t max_pairs) {
  return sdgr_batch_workspace_bytes(n, max_pairs, 1);
}

size_t sdgr_batch_workspace_bytes(int64_t n, int64_t max_pairs, int n_views) {
  if (n_views < 1 || n_views > SDGR_MAX_BATCH) return 0;
  return batch_ws_bytes(n < 1 ? 1 : n, max_pairs < 1 ? 1 : max_pairs, n_views);
}

int sdgr_project(const sdgr_scene* scene, const sdgr_view* view, sdgr_projection* proj, void* stream) {
  return sdgr_project_batch(scene, 1, view, proj, stream);
}

int sdgr_project_batch(const sdgr_scene* scene, int n_views, const sdgr_view* views, sdgr_projection* projs,
                       void* stream) {
  if (!scene || !projs || !views || n_views < 1 || n_views > SDGR_MAX_BATCH) return SDGR_ERR_INVALID;
  if (scene->n < 1 || (scene->dtype != 0 && scene->dtype != 1)) return SDGR_ERR_INVALID;
  for (int k = 0; k < n_views; ++k)
    if (!view_ok(views + k) || projs[k].n != scene->n) return SDGR_ERR_INVALID;
  return launch_project(*scene, n_views, views, projs, static_cast<cudaStream_t>(stream));
}

int sdgr_depth_order(const sdgr_projection* proj, int32_t* order, void* ws, size_t ws_bytes,
                     void* stream) {
  return sdgr_depth_order_batch(1, proj, &order, ws, ws_bytes, stream);
}

int sdgr_depth_order_batch(int n_views, const sdgr_projection* projs, int32_t* const* orders, void* ws,
                           size_t ws_bytes, void* stream) {
  if (n_views < 1 || n_views > SDGR_MAX_BATCH || !projs || !orders || !ws) return SDGR_ERR_INVALID;
  for (int k = 0; k < n_views; ++k)
    if (!orders[k] || projs[k].n < 1 || projs[k].n != projs[0].n) return SDGR_ERR_INVALID;
  return launch_depth_order_batch(n_views, projs, orders, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

int sdgr_count_pairs(const sdgr_projection* proj, int32_t plane, const int32_t* order,
                     int32_t* offsets, void* ws, size_t ws_bytes, void* stream) {
  if (!proj || !offsets || !ws || proj->n < 1 || (plane != 0 && plane != 1)) return SDGR_ERR_INVALID;
  const sdgr_plane& pl = plane == 0 ? proj->comp : proj->img;
  const int32_t* nt = pl.n_tiles;
  return launch_count_batch(1, &nt, &order, proj->n, &offsets, ws, ws_bytes, static_cast<cudaStream_t>(stream));
}

static bool bin_args_ok(const sdgr_projection* proj, const sdgr_view* view, const int32_t* order,
                        const int32_t* offsets, const sdgr_tiles* tiles) {
  if (!proj || !view_ok(view) || !offsets || !tiles_ok(tiles)) return false;
  if (tiles->plane == 0 && !order) return false;
  if (!tiles->pair_start) return false;
  if (tiles->n_pairs > 0 && (!tiles->pair_tile || !tiles->pair_prim || !tiles->pair_pos || !tiles->pre_prim))
    return false;
  return true;
}

int sdgr_bin_pairs(const sdgr_projection* proj, const sdgr_view* view, const int32_t* order,
                   const int32_t* offsets, sdgr_tiles* tiles, void* ws, size_t ws_bytes,
                   void* stream) {
  if (!ws || !bin_args_ok(proj, view, order, offsets, tiles)) return SDGR_ERR_INVALID;
  if (tiles->n_pairs > 0x7fffffffLL) return SDGR_ERR_CAPACITY;
  const int32_t* ord = tiles->plane == 0 ? order : nullptr;
  int32_t* off = const_cast<int32_t*>(offsets);  // read only: counting is off
  return launch_bin_batch(1, proj, view, tiles->plane, &ord, &off, tiles, false, ws, ws_bytes,
                          static_cast<cudaStream_t>(stream));
}

int sdgr_bin_batch(int n_views, const sdgr_projection* projs, const sdgr_view* views, int32_t plane,
                   const int32_t* const* orders, int32_t* const* offsets, sdgr_tiles* tiles, void* ws,
                   size_t ws_bytes, void* stream) {
  if (n_views < 1 || n_views > SDGR_MAX_BATCH || !projs || !views || !offsets || !tiles || !ws ||
      (plane != 0 && plane != 1) || (plane == 0 && !orders))
    return SDGR_ERR_INVALID;
  for (int k = 0; k < n_views; ++k) {
    if (tiles[k].plane != plane || !bin_args_ok(projs + k, views + k, orders ? orders[k] : nullptr, offsets[k],
                                                tiles + k))
      return SDGR_ERR_INVALID;
    if (tiles[k].n_pairs > 0x7fffffffLL) return SDGR_ERR_CAPACITY;
  }
  return launch_bin_batch(n_views, projs, views, plane, plane == 0 ? orders : nullptr, offsets, tiles, true, ws,
                          ws_bytes, static_cast<cudaStream_t>(stream));
}

int sdgr_composite_forward(const sdgr_view* view, const sdgr_projection* proj, const sdgr_tiles* comp,
                           double s_stop, double* seg_sum, double* seg_base, double* partial_I,
                           double* intensity, int32_t* status, sdgr_replay* replay, void* stream) {
  if (!view_ok(view) || !proj || !tiles_ok(comp) || comp->plane != 0 || !intensity || !status ||
      !comp->pair_start || !replay_ok(replay))
    return SDGR_ERR_INVALID;
  if (comp->n_pairs > 0 && (!seg_sum || !seg_base || !partial_I || !comp->pair_pos || !comp->pair_rec))
    return SDGR_ERR_INVALID;
  if (std::isnan(s_stop)) return SDGR_ERR_INVALID;
  return launch_composite_forward(*view, *proj, *comp, s_stop, seg_sum, seg_base, partial_I, intensity,
                                  status, replay, static_cast<cudaStream_t>(stream));
}

int sdgr_splat(const sdgr_view* view, const sdgr_projection* proj, const double* intensity, void* scratch,
               double* image, void* stream) {
  if (!view_ok(view) || !proj || !intensity || !image || !scratch) return SDGR_ERR_INVALID;
  if (!proj->img.uv || !proj->img.inv_cov || !proj->img.bbox || !proj->img.cell_mask) return SDGR_ERR_INVALID;
  return launch_splat(*view, *proj, intensity, static_cast<double*>(scratch), image,
                      static_cast<cudaStream_t>(stream));
}

int sdgr_grad_image(const sdgr_view* view, const sdgr_projection* proj, const double* intensity,
                    const double* dL_dS, double* acc_img, void* stream) {
  if (!view_ok(view) || !proj || !intensity || !dL_dS || !acc_img) return SDGR_ERR_INVALID;
  return launch_grad_image(*view, *proj, intensity, dL_dS, acc_img, static_cast<cudaStream_t>(stream));
}

int sdgr_grad_intensity(const sdgr_view* view, const sdgr_projection* proj, const sdgr_tiles* comp,
                        double s_stop, const double* seg_base, const double* dL_dI, double* seg_g,
                        double* seg_d, double* partial_g, const sdgr_replay* replay, void* stream) {
  if (!view_ok(view) || !proj || !tiles_ok(comp) || comp->plane != 0 || !dL_dI || !replay_ok(replay))
    return SDGR_ERR_INVALID;
  if (comp->n_pairs > 0 && (!seg_base || !seg_g || !seg_d || !partial_g || !comp->pair_rec))
    return SDGR_ERR_INVALID;
  if (std::isnan(s_stop)) return SDGR_ERR_INVALID;
  return launch_grad_intensity(*view, *proj, *comp, s_stop, seg_base, dL_dI, seg_g, seg_d, partial_g, replay,
                               static_cast<cudaStream_t>(stream));
}

int sdgr_grad_geometry(const sdgr_scene* scene, const sdgr_view* view, const sdgr_projection* proj,
                       const sdgr_tiles* comp, const double* acc_img, const double* partial_g,
                       sdgr_grads* out, int accumulate, void* stream) {
  return sdgr_grad_geometry_batch(scene, 1, view, proj, comp, &acc_img, &partial_g, out, accumulate, stream);
}

int sdgr_grad_geometry_batch(const sdgr_scene* scene, int n_views, const sdgr_view* views,
                             const sdgr_projection* projs, const sdgr_tiles* comps,
                             const double* const* acc_imgs, const double* const* partial_gs,
                             sdgr_grads* out, int accumulate, void* stream) {
  if (!scene || n_views < 1 || n_views > SDGR_MAX_BATCH || !views || !projs || !comps || !acc_imgs ||
      !partial_gs || !out)
    return SDGR_ERR_INVALID;
  for (int k = 0; k < n_views; ++k) {
    const sdgr_tiles* c = comps + k;
    if (!view_ok(views + k) || c->plane != 0 || !c->pair_start || !acc_imgs[k]) return SDGR_ERR_INVALID;
    if (c->n_pairs > 0 && !partial_gs[k]) return SDGR_ERR_INVALID;
    if (scene->n != projs[k].n) return SDGR_ERR_STATE;
  }
  return launch_grad_geometry(*scene, n_views, views, projs, comps, acc_imgs, partial_gs, *out, accumulate,
                              static_cast<cudaStream_t>(stream));
}

int sdgr_cell_pairs(const sdgr_projection* proj, const sdgr_view* view, const sdgr_tiles* tiles,
                    int64_t* offsets, int32_t* prim, double* delta, double* q, double* w, void* stream) {
  if (!proj || !view_ok(view) || !tiles || !offsets || (tiles->plane != 0 && tiles->plane != 1)) return SDGR_ERR_INVALID;
  if (!tiles->pair_prim || !tiles->tile_range || tiles->n_tiles < 1) return SDGR_ERR_INVALID;
  const sdgr_plane& pl = tiles->plane == 0 ? proj->comp : proj->img;
  if (!pl.uv || !pl.inv_cov || !pl.bbox || !pl.cell_mask) return SDGR_ERR_INVALID;   // needs the SoA records
  if (prim && (!delta || !q || !w)) return SDGR_ERR_INVALID;
  return launch_cell_pairs(*proj, *view, *tiles, offsets, prim, delta, q, w, static_cast<cudaStream_t>(stream));
}

int sdgr_exp_check(int64_t n, const double* x, double* y, void* stream) {
  if (n < 0 || (n > 0 && (!x || !y))) return -SDGR_ERR_INVALID;
  return -launch_exp_check(n, x, y, (cudaStream_t)stream);
}

int sdgr_cell_intensities(const sdgr_projection* proj, int64_t n_cells, const int64_t* offsets, const int32_t* prim,
                          const double* w, double* tau, double* trans, double* absorb, double* contrib,
                          void* stream) {
  if (!proj || !proj->kappa || !proj->phase || n_cells < 0 || !offsets || !tau || !trans || !absorb || !contrib)
    return SDGR_ERR_INVALID;
  if (n_cells == 0) return SDGR_OK;
  if (!prim || !w) return SDGR_ERR_INVALID;
  return launch_cell_intensities(*proj, n_cells, offsets, prim, w, tau, trans, absorb, contrib,
                                 static_cast<cudaStream_t>(stream));
}

int sdgr_splat_pair_grads(int64_t n_pairs, const int32_t* pair_pixel, const int32_t* pair_prim, const double* dL_dS,
                          const double* intensity, double* dL_dbeta, void* stream) {
  if (n_pairs < 0) return SDGR_ERR_INVALID;
  if (n_pairs > 0 && (!pair_pixel || !pair_prim || !dL_dS || !intensity || !dL_dbeta)) return SDGR_ERR_INVALID;
  return launch_splat_pair_grads(n_pairs, pair_pixel, pair_prim, dL_dS, intensity, dL_dbeta,
                                 static_cast<cudaStream_t>(stream));
}

int sdgr_stage_grads(const sdgr_projection* proj, int32_t plane, const sdgr_tiles* comp, const double* src,
                     double* out, void* stream) {
  if (!proj || proj->n < 1 || !src || !out || (plane != 0 && plane != 1)) return SDGR_ERR_INVALID;
  if (plane == 0 && (!comp || comp->plane != 0 || !comp->pair_start)) return SDGR_ERR_INVALID;
  return launch_stage_grads(*proj, plane, plane == 0 ? comp : nullptr, src, out, static_cast<cudaStream_t>(stream));
}

int sdgr_grad_geometry_explicit(const sdgr_scene* scene, const sdgr_view* view, const sdgr_projection* proj,
                                const double* ex, sdgr_grads* out, void* stream) {
  if (!scene || !view_ok(view) || !proj || !ex || !out) return SDGR_ERR_INVALID;
  if (scene->n != proj->n) return SDGR_ERR_STATE;
  return launch_grad_geometry_explicit(*scene, *view, *proj, ex, *out, static_cast<cudaStream_t>(stream));
}

int sdgr_project_planes(const sdgr_view* view, int64_t n, const double* uv_comp, const double* uv_img,
                        const double* depth, const double* cov_comp, const double* cov_img, const double* phase_raw,
                        const double* kappa, sdgr_projection* proj, void* stream) {
  if (!view_ok(view) || n < 1 || !uv_comp || !uv_img || !depth || !cov_comp || !cov_img || !phase_raw || !kappa ||
      !proj || proj->n != n)
    return SDGR_ERR_INVALID;
  return launch_project_planes(*view, n, uv_comp, uv_img, depth, cov_comp, cov_img, phase_raw, kappa, *proj,
                               static_cast<cudaStream_t>(stream));
}

size_t sdgr_loss_scratch_bytes(int h, int w) { return h > 0 && w > 0 ? loss_scratch_bytes(h, w) : 0; }

int sdgr_loss(const double* S, const double* Y, int h, int w, double lambda_ssim, double max_val,
              const double* kernel11, double* value, double* dL_dS, void* scratch, void* stream) {
  if (!S || !Y || !value || !dL_dS || !scratch || h < 1 || w < 1) return SDGR_ERR_INVALID;
  if (!(lambda_ssim >= 0.0 && lambda_ssim <= 1.0) || !(max_val > 0.0)) return SDGR_ERR_INVALID;
  if (lambda_ssim > 0.0 && h >= 11 && w >= 11 && !kernel11) return SDGR_ERR_INVALID;
  return launch_loss(S, Y, h, w, lambda_ssim, max_val, kernel11, value, dL_dS, scratch,
                     static_cast<cudaStream_t>(stream));
}

static bool scene_ok(const sdgr_scene* s) {
  return s && s->n >= 1 && (s->dtype == 0 || s->dtype == 1) && s->positions && s->rotations && s->log_scales &&
         s->sh_coeffs && s->ke_raw;
}

int sdgr_adam_step(sdgr_scene* scene, const sdgr_grads* grads, sdgr_scene* m, sdgr_scene* v, const double* lr,
                   double beta1, double beta2, double eps, double bc1, double bc2, double displacement_bound,
                   unsigned long long* n_skipped, const int32_t* guard, void* stream) {
  if (!scene_ok(scene) || !scene_ok(m) || !scene_ok(v) || !grads || !lr || !n_skipped) return SDGR_ERR_INVALID;
  if (grads->dtype != 0) return SDGR_ERR_INVALID;
  if (m->n != scene->n || v->n != scene->n || m->dtype != scene->dtype || v->dtype != scene->dtype)
    return SDGR_ERR_STATE;
  if (!grads->positions || !grads->rotations || !grads->log_scales || !grads->sh_coeffs || !grads->ke_raw)
    return SDGR_ERR_INVALID;
  if (!(bc1 > 0.0) || !(bc2 > 0.0)) return SDGR_ERR_INVALID;
  return launch_adam(*scene, *grads, *m, *v, lr, beta1, beta2, eps, bc1, bc2, displacement_bound, n_skipped,
                     guard, static_cast<cudaStream_t>(stream));
}

int sdgr_accum_update(const sdgr_grads* grads, int64_t n, double* norm_sum, double* pos_sum, double* count,
                      void* stream) {
  if (!grads || n < 0 || !norm_sum || !pos_sum || !count || !grads->positions || !grads->uv_grad_norm ||
      !grads->visible || grads->dtype != 0)
    return SDGR_ERR_INVALID;
  if (n == 0) return SDGR_OK;
  return launch_accum_update(*grads, n, norm_sum, pos_sum, count, static_cast<cudaStream_t>(stream));
}

int sdgr_densify_flags(const sdgr_scene* scene, const double* norm_sum, const double* count, double cap,
                       double small_size, double grad_thr, uint8_t* flags, void* stream) {
  if (!scene_ok(scene) || !norm_sum || !count || !flags) return SDGR_ERR_INVALID;
  return launch_densify_flags(*scene, norm_sum, count, cap, small_size, grad_thr, flags,
                              static_cast<cudaStream_t>(stream));
}

int sdgr_clone_shift(sdgr_scene* clones, const double* pos_sum, const double* count, double position_lr,
                     void* stream) {
  if (!clones || clones->n < 0 || !pos_sum || !count) return SDGR_ERR_INVALID;
  if (clones->n == 0) return SDGR_OK;
  if (!scene_ok(clones)) return SDGR_ERR_INVALID;
  return launch_clone_shift(*clones, pos_sum, count, position_lr, static_cast<cudaStream_t>(stream));
}

int sdgr_split_children(sdgr_scene* children, const double* xi, double log_shrink, void* stream) {
  if (!children || children->n < 0 || !xi) return SDGR_ERR_INVALID;
  if (children->n == 0) return SDGR_OK;
  if (!scene_ok(children)) return SDGR_ERR_INVALID;
  return launch_split_children(*children, xi, log_shrink, static_cast<cudaStream_t>(stream));
}

int sdgr_prune_flags(const sdgr_scene* scene, double cap, double phase_floor, uint8_t* survive, void* stream) {
  if (!scene_ok(scene) || !survive) return SDGR_ERR_INVALID;
  return launch_prune_flags(*scene, cap, phase_floor, 0.28209479177387814, survive,
                            static_cast<cudaStream_t>(stream));
}

int sdgr_ply_pack(const sdgr_scene* scene, double* out, void* stream) {
  if (!scene || scene->n < 0 || !out) return SDGR_ERR_INVALID;
  if (scene->n == 0) return SDGR_OK;
  if (!scene_ok(scene)) return SDGR_ERR_INVALID;
  return launch_ply_pack(*scene, out, static_cast<cudaStream_t>(stream));
}

int sdgr_ply_unpack(const double* in, int64_t n, int stride, const int32_t* col, sdgr_scene* scene, void* stream) {
  if (!scene || !col || n < 0 || stride < 28 || scene->n != n) return SDGR_ERR_INVALID;
  if (n == 0) return SDGR_OK;
  if (!in || !scene_ok(scene)) return SDGR_ERR_INVALID;
  for (int k = 0; k < 28; ++k)
    if (col[k] < 0 || col[k] >= stride) return SDGR_ERR_INVALID;
  return launch_ply_unpack(in, n, stride, col, *scene, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
