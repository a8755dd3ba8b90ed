// composite.cu — K6/K7/K9: the tile walks.
//
// A work item is one depth segment (<= seg_len Gaussians) of one 16x16 tile
// list.  A persistent CTA of 256 threads pulls items from an atomic counter;
// thread r owns ray (cell / pixel) r of the tile.  The segment is processed in
// chunks of 256 Gaussians:
//   1. thread j stages Gaussian j (center, inverse covariance, kappa, P, ...)
//      in shared memory and derives its 256-bit in-tile member mask from the
//      8x8 cell window K1 stored (the exact FP64 membership decision is
//      reused, never recomputed); it ORs bit j into the rows of the
//      cell-major 256x256 membership bitmap;
//   2. thread r walks the set bits of its cell's row in ascending order --
//      exactly its ray's member list in (depth, index) order -- and applies
//      the mode's per-pair update in FP64;
//   3. (kContrib, kGrad) per-pair values go to a shared-memory pool at a slot
//      fixed by the Gaussian's member mask; thread j then reduces its own
//      slots in cell order and writes ONE partial record per (tile, Gaussian)
//      pair, indexed by the pair's pre-sort position.  No atomics on the
//      common path and a fixed summation order: results are deterministic.
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
constexpr int kPool = 4096;  // pooled per-pair values per chunk

struct WalkArgs {
  sdgr_plane pl;
  int n_cols, n_rows, tiles_x;
  double cutoff;
  const int32_t* pair_prim;
  const int32_t* pair_pos;
  const int32_t* items;
  const int32_t* n_items;
  uint32_t* counter;
  const double* kappa;
  const double* phase;
  const double* gvec;      // kSplat: intensity; kGSum/kGrad: dL/dI
  double s_stop;
  const double* seg_base;  // exclusive prefix of optical depth per (item, ray)
  const double* seg_g;     // kGrad: this segment's sum of g*contrib
  const double* seg_d;     // kGrad: downstream (later segments) sum of g*contrib
  double* seg_out;         // kSum: seg sums; kSplat: partial pixels; kGSum: seg_g
  double* partial;         // kContrib: (n_pairs); kGrad: (n_pairs, 8)
  int32_t* status;
};

// 256-bit in-tile member mask of one Gaussian (bit = local cell (iv&15)*16+(iu&15)).
__device__ __forceinline__ void member_mask(short4 bb, uint64_t cm, double2 uv, double4 A, int tx,
                                            int ty, double cutoff, uint64_t m[4]) {
  m[0] = m[1] = m[2] = m[3] = 0;
  if ((bb.y - bb.x) < 8 && (bb.w - bb.z) < 8) {
    while (cm) {
      const int b = __ffsll((long long)cm) - 1;
      cm &= cm - 1;
      const int iu = bb.x + (b & 7), iv = bb.z + (b >> 3);
      if ((iu >> 4) == tx && (iv >> 4) == ty) {
        const int c = ((iv & 15) << 4) | (iu & 15);
        const uint64_t bit = 1ull << (c & 63);
#pragma unroll
        for (int w = 0; w < 4; ++w) m[w] |= (c >> 6) == w ? bit : 0ull;
      }
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
      if (member) {
        const int c = ((iv & 15) << 4) | (iu & 15);
        const uint64_t bit = 1ull << (c & 63);
#pragma unroll
        for (int w = 0; w < 4; ++w) m[w] |= (c >> 6) == w ? bit : 0ull;
      }
    }
  }
}

__device__ __forceinline__ int block_excl_scan_i32(int x, int32_t* tmp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int s = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, s, off);
    if (lane >= off) s += y;
  }
  if (lane == 31) tmp[warp] = s;
  __syncthreads();
  int pre = 0;
  for (int w = 0; w < warp; ++w) pre += tmp[w];
  __syncthreads();
  return pre + s - x;
}

// Gradient terms of one computation-plane pair (backward.py:122-148) given
// y1 = T (1 - a) and y2 = dL/dtau * w; accumulated into r[0..6].
__device__ __forceinline__ void grad_terms(double y1, double y2, double kap, double dx, double dy,
                                           double a00, double a01, double a11, double* r) {
  const double dq = -kap * y2;
  r[0] += y1;
  r[1] += y2;
  r[2] += dq * dx * dx;
  r[3] += dq * dx * dy;
  r[4] += dq * dy * dy;
  r[5] += -2.0 * dq * (a00 * dx + a01 * dy);
  r[6] += -2.0 * dq * (a01 * dx + a11 * dy);
}

template <int MODE>
__global__ void __launch_bounds__(256) k_walk(WalkArgs a) {
  constexpr bool kPooled = MODE == kContrib || MODE == kGrad;
  constexpr int kVals = MODE == kGrad ? 2 : 1;
  constexpr int kGW = kPooled ? kChunk : 1;
  __shared__ uint32_t cellbits[8 * kRays];
  __shared__ uint64_t gbits[4 * kGW];
  __shared__ uint32_t gpre[kGW];
  __shared__ int32_t pool_off[kGW];
  __shared__ int32_t spos[kGW];
  __shared__ double su[kChunk], sv[kChunk], sa0[kChunk], sa1[kChunk], sa2[kChunk];
  __shared__ double sk[kChunk], sp[kChunk], sg[kChunk];
  __shared__ int32_t scan_tmp[8];
  __shared__ int item_s;
  extern __shared__ double pool[];

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
    const int64_t slot_ray = (int64_t)item * kRays + tid;
    double S = 0.0, accd = 0.0, rem = 0.0;
    if (MODE == kContrib || MODE == kGSum || MODE == kGrad) S = a.seg_base[slot_ray];
    if (MODE == kGrad) rem = a.seg_d[slot_ray] + a.seg_g[slot_ray];
    bool alive = valid && (MODE == kSplat || S < a.s_stop);
    bool bad = false;
    const int rw = tid >> 6;
    const uint64_t rlow = (1ull << (tid & 63)) - 1ull;

    int cs = start;
    for (; cs < end; cs += kChunk) {
      if (!__syncthreads_or(alive)) break;
#pragma unroll
      for (int w = 0; w < 8; ++w) cellbits[w * kRays + tid] = 0u;
      const int idx = cs + tid;
      const bool have = idx < end;
      uint64_t gm[4] = {0, 0, 0, 0};
      int pos = 0;
      if (have) {
        const int g = a.pair_prim[idx];
        const double2 uv = reinterpret_cast<const double2*>(a.pl.uv)[g];
        const double4 A = reinterpret_cast<const double4*>(a.pl.inv_cov)[g];
        const short4 bb = reinterpret_cast<const short4*>(a.pl.bbox)[g];
        member_mask(bb, a.pl.cell_mask[g], uv, A, tx, ty, a.cutoff, gm);
        su[tid] = uv.x; sv[tid] = uv.y;
        sa0[tid] = A.x; sa1[tid] = A.y; sa2[tid] = A.z;
        if (MODE != kSplat) { sk[tid] = a.kappa[g]; sp[tid] = a.phase[g]; }
        if (MODE == kSplat || MODE == kGSum || MODE == kGrad) sg[tid] = a.gvec[g];
        if (kPooled) {
          pos = a.pair_pos[idx];
          spos[tid] = pos;
          const int c0 = __popcll(gm[0]), c1 = __popcll(gm[1]), c2 = __popcll(gm[2]);
#pragma unroll
          for (int w = 0; w < 4; ++w) gbits[w * kGW + tid] = gm[w];
          gpre[tid] = (uint32_t)c0 << 8 | (uint32_t)(c0 + c1) << 16 | (uint32_t)(c0 + c1 + c2) << 24;
        }
      }
      __syncthreads();
      // scatter this Gaussian into the cell-major bitmap
      {
        const uint32_t bit = 1u << (tid & 31);
        uint32_t* col = cellbits + (tid >> 5) * kRays;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          uint64_t m = gm[w];
          while (m) {
            const int b = __ffsll((long long)m) - 1;
            m &= m - 1;
            atomicOr(col + (w * 64 + b), bit);
          }
        }
      }
      int cnt = 0, off = 0;
      if (kPooled) {
        cnt = __popcll(gm[0]) + __popcll(gm[1]) + __popcll(gm[2]) + __popcll(gm[3]);
        off = block_excl_scan_i32(cnt, scan_tmp);
        pool_off[tid] = off;
        for (int k = off; k < min(off + cnt, kPool); ++k)
#pragma unroll
          for (int v = 0; v < kVals; ++v) pool[k * kVals + v] = 0.0;
        if (have && off + cnt > kPool) {  // overflow: ray threads add into the record
          if (MODE == kContrib) a.partial[pos] = 0.0;
          else
#pragma unroll
            for (int k = 0; k < 8; ++k) a.partial[(int64_t)pos * 8 + k] = 0.0;
        }
      }
      __syncthreads();
      if (alive) {
#pragma unroll 1
        for (int w = 0; w < 8 && alive; ++w) {
          uint32_t bits = cellbits[w * kRays + tid];
          while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const int jj = w * 32 + b;
            const double dx = dsub(du, su[jj]), dy = dsub(dv, sv[jj]);
            const double q = quadform(sa0[jj], sa1[jj], sa2[jj], dx, dy);
            const double wgt = exp(-q);
            if (MODE == kSplat) {
              accd += wgt * sg[jj];
              continue;
            }
            const double tau = sk[jj] * wgt;
            if (MODE == kSum) {
              S += tau;
              if (S > a.s_stop) { alive = false; break; }
              continue;
            }
            if (!(S < a.s_stop)) { alive = false; break; }
            const double T = exp(-S);
            const double oma = -expm1(-tau);
            const double P = sp[jj];
            const double c = T * oma * P;
            int slot = 0;
            if (kPooled)
              slot = pool_off[jj] + (int)((gpre[jj] >> (8 * rw)) & 255u) +
                     __popcll(gbits[rw * kGW + jj] & rlow);
            if (MODE == kContrib) {
              if (!isfinite(c)) bad = true;
              if (slot < kPool) pool[slot] = c;
              else atomicAdd(a.partial + spos[jj], c);
            } else if (MODE == kGSum) {
              accd += sg[jj] * c;
            } else {  // kGrad
              const double gI = sg[jj];
              rem -= gI * c;  // downstream sum of g*contrib after this pair
              const double dtau = gI * T * exp(-tau) * P - rem;
              const double y1 = T * oma, y2 = dtau * wgt;
              if (slot < kPool) {
                pool[2 * slot] = y1;
                pool[2 * slot + 1] = y2;
              } else {
                double r[7] = {0, 0, 0, 0, 0, 0, 0};
                grad_terms(y1, y2, sk[jj], dx, dy, sa0[jj], sa1[jj], sa2[jj], r);
                r[0] *= gI;
                double* rec = a.partial + (int64_t)spos[jj] * 8;
#pragma unroll
                for (int k = 0; k < 7; ++k) atomicAdd(rec + k, r[k]);
              }
            }
            S += tau;
          }
        }
      }
      if (kPooled) {
        __syncthreads();
        if (have) {
          // reduce this Gaussian's pooled pairs in ascending cell order
          double r[7] = {0, 0, 0, 0, 0, 0, 0};
          int k = off;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            uint64_t m = gm[w];
            while (m && k < kPool) {
              const int b = __ffsll((long long)m) - 1;
              m &= m - 1;
              if (MODE == kContrib) {
                r[0] += pool[k];
              } else {
                const int c = w * 64 + b;
                const double dx = dsub((double)(tx * kTile + (c & 15)), su[tid]);
                const double dy = dsub((double)(ty * kTile + (c >> 4)), sv[tid]);
                grad_terms(pool[2 * k], pool[2 * k + 1], sk[tid], dx, dy, sa0[tid], sa1[tid], sa2[tid], r);
              }
              ++k;
            }
          }
          if (MODE == kContrib) {
            if (off + cnt > kPool) atomicAdd(a.partial + pos, r[0]);
            else a.partial[pos] = r[0];
          } else {
            r[0] *= sg[tid];
            double* rec = a.partial + (int64_t)pos * 8;
            if (off + cnt > kPool) {
#pragma unroll
              for (int q = 0; q < 7; ++q) atomicAdd(rec + q, r[q]);
            } else {
              reinterpret_cast<double4*>(rec)[0] = make_double4(r[0], r[1], r[2], r[3]);
              reinterpret_cast<double4*>(rec)[1] = make_double4(r[4], r[5], r[6], 0.0);
            }
          }
        }
      }
    }
    // every Gaussian of the segment owns a record: zero the ones past an early exit
    if (kPooled) {
      for (int i = cs + tid; i < end; i += kChunk) {
        const int p = a.pair_pos[i];
        if (MODE == kContrib) a.partial[p] = 0.0;
        else {
          double4* rec = reinterpret_cast<double4*>(a.partial + (int64_t)p * 8);
          rec[0] = make_double4(0, 0, 0, 0);
          rec[1] = make_double4(0, 0, 0, 0);
        }
      }
    }
    if (MODE == kSum) a.seg_out[slot_ray] = S;
    if (MODE == kSplat || MODE == kGSum) a.seg_out[slot_ray] = accd;
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
                                                      const double* part, double* image) {
  const int t = blockIdx.x;
  const int iu = (t % tiles_x) * kTile + (threadIdx.x & 15);
  const int iv = (t / tiles_x) * kTile + (threadIdx.x >> 4);
  if (iu >= n_az || iv >= n_rg) return;
  const int cnt = range[2 * t + 1] - range[2 * t];
  const int nseg = (cnt + seg_len - 1) / seg_len;
  double s = 0.0;
  const int64_t first = nseg ? tile_first[t] : 0;
  for (int k = 0; k < nseg; ++k) s += part[(first + k) * kRays + threadIdx.x];
  image[(int64_t)iv * n_az + iu] = s;
}

// intensity[g] = sum of its per-tile partials, in pre-sort (tile-id) order.
__global__ void __launch_bounds__(256) k_reduce_intensity(const int32_t* pair_start, const int32_t* n_tiles,
                                                          const double* partial, int64_t n, double* out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  const int s = pair_start[g], c = n_tiles[g];
  double acc = 0.0;
  for (int k = 0; k < c; ++k) acc += partial[s + k];
  out[g] = acc;
}

template <int MODE>
static int walk_grid(int max_items, size_t smem) {
  static int per_sm = 0;
  static int sms = 0;
  if (per_sm == 0) {
    if (smem > 0)
      cudaFuncSetAttribute(k_walk<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_walk<MODE>, 256, smem);
    per_sm = b > 0 ? b : 1;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return max(1, min(max_items, sms * per_sm));
}

template <int MODE>
static int launch_walk(const WalkArgs& a, int max_items, cudaStream_t st) {
  constexpr size_t smem = MODE == kGrad ? 2 * kPool * sizeof(double)
                                        : (MODE == kContrib ? kPool * sizeof(double) : 0);
  if (cudaMemsetAsync(a.counter, 0, sizeof(uint32_t), st) != cudaSuccess) return SDGR_ERR_CUDA;
  k_walk<MODE><<<walk_grid<MODE>(max_items, smem), 256, smem, st>>>(a);
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
  a.pair_pos = t.pair_pos;
  a.items = t.items;
  a.n_items = t.n_items;
  a.counter = reinterpret_cast<uint32_t*>(t.n_items + 2);
  a.kappa = p.kappa;
  a.phase = p.phase;
  return a;
}

int launch_composite_forward(const sdgr_view& v, const sdgr_projection& p, const sdgr_tiles& t,
                             double s_stop, double* seg_sum, double* seg_base, double* partial_I,
                             double* intensity, int32_t* status, cudaStream_t st) {
  if (t.n_pairs > 0) {
    WalkArgs a = base_args(v, p, t);
    a.s_stop = s_stop;
    a.seg_out = seg_sum;
    int rc = launch_walk<kSum>(a, t.max_items, st);
    if (rc) return rc;
    k_seg_scan<false><<<t.n_tiles, 256, 0, st>>>(t.tile_range, t.tile_first, t.seg_len, seg_sum, seg_base);
    note_launch();
    a.seg_base = seg_base;
    a.seg_out = nullptr;
    a.partial = partial_I;
    a.status = status;
    rc = launch_walk<kContrib>(a, t.max_items, st);
    if (rc) return rc;
  }
  k_reduce_intensity<<<(unsigned)((p.n + 255) / 256), 256, 0, st>>>(t.pair_start, p.comp.n_tiles, partial_I,
                                                                     p.n, intensity);
  note_launch();
  return check_launch();
}

int launch_splat(const sdgr_view& v, const sdgr_projection& p, const sdgr_tiles& t,
                 const double* intensity, double* part, double* image, cudaStream_t st) {
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
                          double s_stop, const double* seg_base, const double* dL_dI, double* seg_g,
                          double* seg_d, double* partial_g, cudaStream_t st) {
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
  a.partial = partial_g;
  return launch_walk<kGrad>(a, t.max_items, st);
}

}  // namespace sdgr
