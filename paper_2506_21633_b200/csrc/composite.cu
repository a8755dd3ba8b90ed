// composite.cu — K6/K7/K9: the tile walks.
//
// A work item is one depth segment (<= seg_len Gaussians) of one 16x16 tile
// list.  A persistent CTA of 256 threads pulls items from an atomic counter;
// thread r owns ray (cell / pixel) r of the tile.  The segment is processed in
// chunks of 256 Gaussians:
//   1. thread j stages Gaussian j (center, inverse covariance, kappa, P, ...)
//      in shared memory and ORs bit j into the 256x256 membership bitmap of
//      every tile cell its footprint covers (cell bit-window from K1, so the
//      exact FP64 membership decision is reused, never recomputed);
//   2. thread r walks the set bits of its cell's row in ascending order --
//      i.e. exactly its ray's member list in (depth, index) order -- and
//      applies the mode's per-pair update;
//   3. per-Gaussian partial sums collected in shared memory are flushed to
//      global memory with one atomic per Gaussian per chunk.
// Only true members are visited: no per-candidate rejection work.
//
// Modes (reference stage they replace):
//   kSum     segment optical-depth sums          (forward.py:182-187, cumsum)
//   kContrib per-pair contributions -> I_g        (forward.py:188-192)
//   kSplat   image = sum_g w I_g per pixel        (forward.py:227-240)
//   kGSum    segment sums of g*contrib            (backward.py:129-139)
//   kGrad    reverse-recurrence gradients         (backward.py:122-148)
// Depth segments are stitched with per-ray exclusive prefix (forward) /
// suffix (backward) scans over a tile's items, in FP64.
//
// Early ray termination: a ray stops once its log-transmittance S exceeds
// s_stop (contributions < e^-s_stop * P).  s_stop = +inf reproduces the
// reference's exhaustive walk.
#include "common.cuh"

namespace sdgr {

enum WalkMode { kSum = 0, kContrib = 1, kSplat = 2, kGSum = 3, kGrad = 4 };

struct WalkArgs {
  sdgr_plane pl;
  int n_cols, n_rows, tiles_x;
  double cutoff;
  const int32_t* pair_prim;
  const int32_t* items;
  const int32_t* n_items;
  uint32_t* counter;
  const float* kappa;
  const float* phase;
  const float* gvec;       // kSplat: intensity; kGSum/kGrad: dL/dI
  double s_stop;
  const double* seg_base;  // exclusive prefix of optical depth per (item, ray)
  const double* seg_g;     // kGrad: this segment's sum of g*contrib
  const double* seg_d;     // kGrad: downstream (later segments) sum of g*contrib
  double* seg_out;         // kSum: seg sums; kSplat: partial pixels; kGSum: seg_g
  float* acc_out;          // kContrib: intensity (n); kGrad: acc (7, n)
  int64_t n;
  int32_t* status;
};

__device__ __forceinline__ void build_mask(uint32_t* mask, int j, short4 bb, uint64_t cm,
                                           double2 uv, double4 A, int tx, int ty, double cutoff) {
  const uint32_t bit = 1u << (j & 31);
  uint32_t* col = mask + (j >> 5) * kRays;
  if ((bb.y - bb.x) < 8 && (bb.w - bb.z) < 8) {
    while (cm) {
      const int b = __ffsll((long long)cm) - 1;
      cm &= cm - 1;
      const int iu = bb.x + (b & 7), iv = bb.z + (b >> 3);
      if ((iu >> 4) == tx && (iv >> 4) == ty) atomicOr(col + (((iv & 15) << 4) | (iu & 15)), bit);
    }
    return;
  }
  // large footprint: exact FP64 test of the bbox cells inside this tile
  const bool dense = !isfinite(cutoff);
  const double cut2 = dmul(cutoff, cutoff), a01x2 = dmul(2.0, A.y);
  const int cx0 = max((int)bb.x, tx * kTile), cx1 = min((int)bb.y, tx * kTile + kTile - 1);
  const int cy0 = max((int)bb.z, ty * kTile), cy1 = min((int)bb.w, ty * kTile + kTile - 1);
  for (int iv = cy0; iv <= cy1; ++iv) {
    const double dy = dsub((double)iv, uv.y);
    const double t3 = dmul(A.z, dmul(dy, dy));
    for (int iu = cx0; iu <= cx1; ++iu) {
      bool member = dense;
      if (!dense) {
        const double dx = dsub((double)iu, uv.x);
        const double q = dadd(dadd(dmul(A.x, dmul(dx, dx)), dmul(dmul(a01x2, dx), dy)), t3);
        member = q <= cut2;
      }
      if (member) atomicOr(col + (((iv & 15) << 4) | (iu & 15)), bit);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_walk(WalkArgs a) {
  constexpr int kAcc = MODE == kContrib ? 1 : (MODE == kGrad ? 7 : 0);
  __shared__ uint32_t mask[8 * kRays];
  __shared__ double su[kChunk], sv[kChunk], sa0[kChunk], sa1[kChunk], sa2[kChunk];
  __shared__ float sk[kChunk], sp[kChunk], sg[kChunk];
  __shared__ float acc[kAcc > 0 ? kAcc : 1][kChunk];
  __shared__ int item_s;
  const int tid = threadIdx.x;
  const int n_items = *a.n_items;
  while (true) {
    __syncthreads();
    if (tid == 0) item_s = (int)atomicAdd(a.counter, 1u);
    __syncthreads();
    const int item = item_s;
    if (item >= n_items) return;
    const int4 it = reinterpret_cast<const int4*>(a.items)[item];
    const int tile = it.x, start = it.y, end = it.z;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int iu = tx * kTile + (tid & 15), iv = ty * kTile + (tid >> 4);
    const bool valid = iu < a.n_cols && iv < a.n_rows;
    const double du = (double)iu, dv = (double)iv;
    const int64_t slot = (int64_t)item * kRays + tid;
    double S = 0.0, accd = 0.0, rem = 0.0;
    if (MODE == kContrib || MODE == kGSum || MODE == kGrad) S = a.seg_base[slot];
    if (MODE == kGrad) rem = a.seg_d[slot] + a.seg_g[slot];
    bool alive = valid && (MODE == kSplat || S < a.s_stop);
    bool bad = false;

    for (int cs = start; cs < end; cs += kChunk) {
      if (!__syncthreads_or(alive)) break;
#pragma unroll
      for (int w = 0; w < 8; ++w) mask[w * kRays + tid] = 0u;
      const int idx = cs + tid;
      const bool have = idx < end;
      int g = 0;
      short4 bb = make_short4(1, 0, 1, 0);
      uint64_t cm = 0;
      double2 uv = make_double2(0.0, 0.0);
      double4 A = make_double4(0.0, 0.0, 0.0, 0.0);
      if (have) {
        g = a.pair_prim[idx];
        uv = reinterpret_cast<const double2*>(a.pl.uv)[g];
        A = reinterpret_cast<const double4*>(a.pl.inv_cov)[g];
        bb = reinterpret_cast<const short4*>(a.pl.bbox)[g];
        cm = a.pl.cell_mask[g];
        su[tid] = uv.x; sv[tid] = uv.y;
        sa0[tid] = A.x; sa1[tid] = A.y; sa2[tid] = A.z;
        if (MODE != kSplat) { sk[tid] = a.kappa[g]; sp[tid] = a.phase[g]; }
        if (MODE == kSplat || MODE == kGSum || MODE == kGrad) sg[tid] = a.gvec[g];
#pragma unroll
        for (int k = 0; k < kAcc; ++k) acc[k][tid] = 0.f;
      }
      __syncthreads();
      if (have) build_mask(mask, tid, bb, cm, uv, A, tx, ty, a.cutoff);
      __syncthreads();
      if (alive) {
#pragma unroll 1
        for (int w = 0; w < 8 && alive; ++w) {
          uint32_t bits = mask[w * kRays + tid];
          while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int jj = w * 32 + b;
            const double dx = dsub(du, su[jj]), dy = dsub(dv, sv[jj]);
            const double q = quadform(sa0[jj], sa1[jj], sa2[jj], dx, dy);
            const float wgt = expf(-(float)q);
            if (MODE == kSplat) {
              accd += (double)wgt * (double)sg[jj];
              continue;
            }
            const float tau = sk[jj] * wgt;
            if (MODE == kSum) {
              S += (double)tau;
              if (S > a.s_stop) { alive = false; break; }
              continue;
            }
            if (!(S < a.s_stop)) { alive = false; break; }
            const float T = expf(-(float)S);
            const float oma = -expm1f(-tau);
            const float P = sp[jj];
            const float c = T * oma * P;
            if (MODE == kContrib) {
              atomicAdd(&acc[0][jj], c);
              if (!isfinite(c)) bad = true;
            } else if (MODE == kGSum) {
              accd += (double)sg[jj] * (double)c;
            } else {  // kGrad
              const float gI = sg[jj];
              rem -= (double)gI * (double)c;        // downstream of this pair
              const float ab = expf(-tau);
              const float dtau = (float)((double)(gI * T * ab * P) - rem);
              const float dq = -dtau * sk[jj] * wgt;
              const float fx = (float)dx, fy = (float)dy;
              atomicAdd(&acc[0][jj], gI * T * oma);
              atomicAdd(&acc[1][jj], dtau * wgt);
              atomicAdd(&acc[2][jj], dq * fx * fx);
              atomicAdd(&acc[3][jj], dq * fx * fy);
              atomicAdd(&acc[4][jj], dq * fy * fy);
              const float ax = (float)(sa0[jj] * dx + sa1[jj] * dy);
              const float ay = (float)(sa1[jj] * dx + sa2[jj] * dy);
              atomicAdd(&acc[5][jj], -2.f * dq * ax);
              atomicAdd(&acc[6][jj], -2.f * dq * ay);
            }
            S += (double)tau;
          }
        }
      }
      __syncthreads();
      if (kAcc > 0 && have) {
#pragma unroll
        for (int k = 0; k < kAcc; ++k) {
          const float v = acc[k][tid];
          if (v != 0.f) atomicAdd(a.acc_out + (int64_t)k * a.n + g, v);
        }
      }
    }
    if (MODE == kSum) a.seg_out[slot] = S;
    if (MODE == kSplat || MODE == kGSum) a.seg_out[slot] = accd;
    if (MODE == kContrib && __syncthreads_or(bad) && tid == 0) atomicOr(a.status + SDGR_STATUS_NONFINITE, 1);
  }
}

// Per-ray exclusive prefix (forward) or suffix (backward) over a tile's
// segment items.  One CTA per tile, thread = ray.
template <bool kSuffix>
__global__ void __launch_bounds__(256) k_seg_scan(const int32_t* range, const int32_t* tile_first,
                                                  int seg_len, const double* in, double* out) {
  const int t = blockIdx.x;
  const int cnt = range[2 * t + 1] - range[2 * t];
  const int nseg = (cnt + seg_len - 1) / seg_len;
  if (nseg == 0) return;
  const int64_t first = tile_first[t];
  double run = 0.0;
  for (int k = 0; k < nseg; ++k) {
    const int64_t s = (first + (kSuffix ? nseg - 1 - k : k)) * kRays + threadIdx.x;
    const double v = in[s];
    out[s] = run;
    run += v;
  }
}

// image[pixel] = sum over the tile's segment partials, in item order.
__global__ void __launch_bounds__(256) k_splat_reduce(const int32_t* range, const int32_t* tile_first,
                                                      int seg_len, int tiles_x, int n_az, int n_rg,
                                                      const double* part, float* image) {
  const int t = blockIdx.x;
  const int iu = (t % tiles_x) * kTile + (threadIdx.x & 15);
  const int iv = (t / tiles_x) * kTile + (threadIdx.x >> 4);
  if (iu >= n_az || iv >= n_rg) return;
  const int cnt = range[2 * t + 1] - range[2 * t];
  const int nseg = (cnt + seg_len - 1) / seg_len;
  double s = 0.0;
  const int64_t first = nseg ? tile_first[t] : 0;
  for (int k = 0; k < nseg; ++k) s += part[(first + k) * kRays + threadIdx.x];
  image[(int64_t)iv * n_az + iu] = (float)s;
}

template <int MODE>
static int walk_grid(int max_items) {
  static int per_sm = 0;
  if (per_sm == 0) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_walk<MODE>, 256, 0);
    per_sm = b > 0 ? b : 1;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int resident = sms * per_sm;
  return max(1, min(max_items, resident));
}

template <int MODE>
static int launch_walk(const WalkArgs& a, int max_items, cudaStream_t st) {
  if (cudaMemsetAsync(a.counter, 0, sizeof(uint32_t), st) != cudaSuccess) return SDGR_ERR_CUDA;
  k_walk<MODE><<<walk_grid<MODE>(max_items), 256, 0, st>>>(a);
  note_launch();
  return check_launch();
}

static WalkArgs base_args(const sdgr_view& v, const sdgr_projection& p, const sdgr_tiles& t) {
  WalkArgs a{};
  a.pl = t.plane == 0 ? p.comp : p.img;
  a.n_cols = t.plane == 0 ? v.n_u : v.n_az;
  a.n_rows = t.plane == 0 ? v.n_v : v.n_rg;
  a.tiles_x = t.tiles_x;
  a.cutoff = v.cutoff;
  a.pair_prim = t.pair_prim;
  a.items = t.items;
  a.n_items = t.n_items;
  a.counter = reinterpret_cast<uint32_t*>(t.n_items + 2);
  a.kappa = p.kappa;
  a.phase = p.phase;
  a.n = p.n;
  return a;
}

int launch_composite_forward(const sdgr_view& v, const sdgr_projection& p, const sdgr_tiles& t,
                             double s_stop, double* seg_sum, double* seg_base, float* intensity,
                             int32_t* status, cudaStream_t st) {
  if (cudaMemsetAsync(intensity, 0, sizeof(float) * p.n, st) != cudaSuccess) return SDGR_ERR_CUDA;
  if (t.n_pairs == 0) return SDGR_OK;
  WalkArgs a = base_args(v, p, t);
  a.s_stop = s_stop;
  a.seg_out = seg_sum;
  int rc = launch_walk<kSum>(a, t.max_items, st);
  if (rc) return rc;
  k_seg_scan<false><<<t.n_tiles, 256, 0, st>>>(t.tile_range, t.tile_first, t.seg_len, seg_sum, seg_base);
  note_launch();
  a.seg_base = seg_base;
  a.seg_out = nullptr;
  a.acc_out = intensity;
  a.status = status;
  return launch_walk<kContrib>(a, t.max_items, st);
}

int launch_splat(const sdgr_view& v, const sdgr_projection& p, const sdgr_tiles& t,
                 const float* intensity, double* part, float* image, cudaStream_t st) {
  if (t.n_pairs > 0) {
    WalkArgs a = base_args(v, p, t);
    a.gvec = intensity;
    a.seg_out = part;
    int rc = launch_walk<kSplat>(a, t.max_items, st);
    if (rc) return rc;
  }
  k_splat_reduce<<<t.n_tiles, 256, 0, st>>>(t.tile_range, t.tile_first, t.seg_len, t.tiles_x, v.n_az,
                                            v.n_rg, part, image);
  note_launch();
  return check_launch();
}

int launch_grad_intensity(const sdgr_view& v, const sdgr_projection& p, const sdgr_tiles& t,
                          double s_stop, const double* seg_base, const float* dL_dI, double* seg_g,
                          double* seg_d, float* acc_comp, cudaStream_t st) {
  if (cudaMemsetAsync(acc_comp, 0, sizeof(float) * 7 * p.n, st) != cudaSuccess) return SDGR_ERR_CUDA;
  if (t.n_pairs == 0) return SDGR_OK;
  WalkArgs a = base_args(v, p, t);
  a.s_stop = s_stop;
  a.seg_base = seg_base;
  a.gvec = dL_dI;
  a.seg_out = seg_g;
  int rc = launch_walk<kGSum>(a, t.max_items, st);
  if (rc) return rc;
  k_seg_scan<true><<<t.n_tiles, 256, 0, st>>>(t.tile_range, t.tile_first, t.seg_len, seg_g, seg_d);
  note_launch();
  a.seg_out = nullptr;
  a.seg_g = seg_g;
  a.seg_d = seg_d;
  a.acc_out = acc_comp;
  return launch_walk<kGrad>(a, t.max_items, st);
}

}  // namespace sdgr
