// composite.cu — K6/K7/K9: the tile walks.
//
// A work item is one depth segment (<= seg_len Gaussians) of one 16x16 tile
// list.  A persistent CTA of 256 threads pulls items from an atomic counter.
// Thread r owns ray (cell / pixel) r of the tile for the order-dependent
// steps; thread j owns Gaussian j of the current chunk of 256.
//
// Per chunk:
//   P0  thread j stages Gaussian j and derives its 256-bit in-tile member
//       mask from the 8x8 cell window K1 stored (the exact FP64 membership is
//       reused, never recomputed); bits go into a cell-major 256x256 bitmap.
//   P1  thread r counts its ray's live members; a block scan lays every
//       (ray, member) pair out in a flat shared array in ray-major,
//       depth-minor order -- exactly the per-ray walk order of the reference.
//   P2  thread j evaluates w = exp(-q) for each of its member cells (pair-
//       parallel, full warps) into the pair's flat slot.
//   P3  thread r runs the order-dependent part over its own slots: only
//       additions (log-transmittance prefix, early ray termination).
//   P4  flat pair-parallel pass: T = e^-S, 1 - e^-tau, contributions.
//   P5  thread r: downstream suffix sums (backward only; additions).
//   P7  thread j reduces its own pairs in cell order into ONE partial record
//       per (tile, Gaussian) pair, indexed by the pair's pre-sort position:
//       no atomics, fixed summation order => deterministic results.
// If a chunk has more live pairs than the flat array holds it is processed
// in sub-chunks of consecutive Gaussians (ray state carries over).
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

template <int MODE>
struct WalkCfg {
  static constexpr int kCap = MODE == kGrad ? 2048 : 4096;            // flat pair slots
  static constexpr bool kS = MODE == kContrib || MODE == kGSum || MODE == kGrad;
  static constexpr bool kJ = kS;                                       // slot -> Gaussian
  static constexpr bool kXY = MODE == kGrad;
  static constexpr size_t kSmem = kCap * (8 + (kS ? 8 : 0) + (kXY ? 16 : 0) + (kJ ? 1 : 0));
};

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

// exclusive block scan (256 threads); also returns the block total
__device__ __forceinline__ int block_scan(int x, int32_t* tmp, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int s = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, s, off);
    if (lane >= off) s += y;
  }
  __syncthreads();
  if (lane == 31) tmp[warp] = s;
  __syncthreads();
  int pre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const int v = tmp[w];
    pre += w < warp ? v : 0;
    tot += v;
  }
  total = tot;
  return pre + s - x;
}

// bits of 32-bit word w that belong to Gaussians [j0, j1)
__device__ __forceinline__ uint32_t range_mask(int w, int j0, int j1) {
  const int lo = max(j0 - 32 * w, 0), hi = min(j1 - 32 * w, 32);
  if (hi <= lo) return 0u;
  const uint32_t upper = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
  return upper & ~((1u << lo) - 1u);
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
  using Cfg = WalkCfg<MODE>;
  constexpr int kCap = Cfg::kCap;
  __shared__ uint32_t rows[8 * kRays];   // rows[w*256 + r]: bit (j&31) of word w = Gaussian j covers ray r
  __shared__ uint32_t wpre[2 * kRays];   // per ray: byte prefix counts of the masked words
  __shared__ int32_t ray_off[kRays];
  __shared__ uint32_t alive_bits[8];
  __shared__ double su[kChunk], sv[kChunk], sa0[kChunk], sa1[kChunk], sa2[kChunk];
  __shared__ double sk[kChunk], sp[kChunk], sg[kChunk];
  __shared__ int32_t scan_tmp[8];
  __shared__ int32_t base_s;
  __shared__ int item_s;
  extern __shared__ double dyn[];
  double* fw = dyn;                                         // w (kSum: tau, kSplat: w*I)
  double* fs = fw + kCap;                                   // S / contrib / g*contrib / D
  double* fx = fs + (Cfg::kS ? kCap : 0);                   // kGrad: g*T*a*P
  double* fy = fx + (Cfg::kXY ? kCap : 0);                  // kGrad: T*(1-a)
  uint8_t* fj = reinterpret_cast<uint8_t*>(fy + (Cfg::kXY ? kCap : 0));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
    const int64_t slot_ray = (int64_t)item * kRays + tid;
    double S = 0.0, accd = 0.0, rem = 0.0;
    if (Cfg::kS) S = a.seg_base[slot_ray];
    if (MODE == kGrad) rem = a.seg_d[slot_ray] + a.seg_g[slot_ray];
    bool alive = valid && (MODE == kSplat || S < a.s_stop);
    bool bad = false;

    int cs = start;
    for (; cs < end; cs += kChunk) {
      if (!__syncthreads_or(alive)) break;
      // ---- P0: stage Gaussian j = tid, build its member mask, scatter bits
#pragma unroll
      for (int w = 0; w < 8; ++w) rows[w * kRays + tid] = 0u;
      const int idx = cs + tid;
      const int nG = min(kChunk, end - cs);
      const bool have = tid < nG;
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
        if (MODE == kContrib || MODE == kGrad) pos = a.pair_pos[idx];
      }
      __syncthreads();
      {
        const uint32_t bit = 1u << lane;
        uint32_t* col = rows + warp * kRays;
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
      double racc[7] = {0, 0, 0, 0, 0, 0, 0};  // P7 accumulators of Gaussian tid
      int j0 = 0;
      while (j0 < nG) {
        // ---- live rays and the sub-chunk [j0, j1) that fits the flat array
        const uint32_t ab = __ballot_sync(0xffffffffu, alive);
        if (lane == 0) alive_bits[warp] = ab;
        __syncthreads();
        uint64_t lm[4];
#pragma unroll
        for (int w = 0; w < 4; ++w)
          lm[w] = gm[w] & ((uint64_t)alive_bits[2 * w] | ((uint64_t)alive_bits[2 * w + 1] << 32));
        const int cnt_g = (have && tid >= j0)
                              ? __popcll(lm[0]) + __popcll(lm[1]) + __popcll(lm[2]) + __popcll(lm[3])
                              : 0;
        int tot_g;
        const int excl_g = block_scan(cnt_g, scan_tmp, tot_g);
        if (tid == j0) base_s = excl_g;
        __syncthreads();
        const bool fits = have && tid >= j0 && (excl_g + cnt_g - base_s) <= kCap;
        const int j1 = j0 + __syncthreads_count(fits);
        // ---- P1: per-ray counts of members in [j0, j1), flat offsets
        int cnt_r = 0;
        uint32_t pre_lo = 0, pre_hi = 0;
        if (alive) {
#pragma unroll
          for (int w = 0; w < 8; ++w) {
            const int c = __popc(rows[w * kRays + tid] & range_mask(w, j0, j1));
            if (w < 4) pre_lo |= (uint32_t)cnt_r << (8 * w);
            else pre_hi |= (uint32_t)cnt_r << (8 * (w - 4));
            cnt_r += c;
          }
        }
        wpre[tid] = pre_lo;
        wpre[kRays + tid] = pre_hi;
        int total;
        const int roff = block_scan(cnt_r, scan_tmp, total);
        ray_off[tid] = roff;
        __syncthreads();
        // ---- P2: Gaussian-parallel weights into the flat slots
        const bool mine = have && tid >= j0 && tid < j1;
        if (mine) {
          const int jw = tid >> 5;
          const uint32_t below = ((1u << lane) - 1u) & range_mask(jw, j0, j1);
          const uint32_t pshift = 8 * (jw & 3);
          const uint32_t* wp = wpre + (jw < 4 ? 0 : kRays);
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            uint64_t m = lm[w];
            while (m) {
              const int b = __ffsll((long long)m) - 1;
              m &= m - 1;
              const int r = w * 64 + b;
              const int p = ray_off[r] + (int)((wp[r] >> pshift) & 255u) + __popc(rows[jw * kRays + r] & below);
              const double dx = dsub((double)(tx * kTile + (r & 15)), su[tid]);
              const double dy = dsub((double)(ty * kTile + (r >> 4)), sv[tid]);
              const double wgt = exp(-quadform(sa0[tid], sa1[tid], sa2[tid], dx, dy));
              if (MODE == kSum) fw[p] = sk[tid] * wgt;
              else if (MODE == kSplat) fw[p] = wgt * sg[tid];
              else fw[p] = wgt;
              if (Cfg::kJ) fj[p] = (uint8_t)tid;
            }
          }
        }
        __syncthreads();
        // ---- P3: ray-serial, additions only
        if (cnt_r > 0) {
          const int p0 = roff, p1 = roff + cnt_r;
          if (MODE == kSum) {
            for (int p = p0; p < p1; ++p) {
              S += fw[p];
              if (S > a.s_stop) { alive = false; break; }
            }
          } else if (MODE == kSplat) {
            for (int p = p0; p < p1; ++p) accd += fw[p];
          } else {
            int p = p0;
            for (; p < p1; ++p) {
              if (!(S < a.s_stop)) break;
              fs[p] = S;
              S += sk[fj[p]] * fw[p];
            }
            for (; p < p1; ++p) fs[p] = __longlong_as_double(0x7ff0000000000000ll);  // dead: T = 0
            alive = S < a.s_stop;
          }
        }
        if (Cfg::kS) {
          __syncthreads();
          // ---- P4: flat pair-parallel transmittance and contributions
          for (int p = tid; p < total; p += kRays) {
            const int j = fj[p];
            const double wgt = fw[p];
            const double tau = sk[j] * wgt;
            const double T = exp(-fs[p]);
            const double oma = -expm1(-tau);
            const double c = T * oma * sp[j];
            if (MODE == kContrib) {
              fs[p] = c;
              if (!isfinite(c)) bad = true;
            } else if (MODE == kGSum) {
              fs[p] = sg[j] * c;
            } else {
              const double gI = sg[j];
              fs[p] = gI * c;
              fx[p] = gI * T * exp(-tau) * sp[j];
              fy[p] = T * oma;
            }
          }
          __syncthreads();
          // ---- P5: ray-serial sums of g*contrib (backward)
          if (MODE == kGSum) {
            for (int p = roff; p < roff + cnt_r; ++p) accd += fs[p];
          } else if (MODE == kGrad) {
            for (int p = roff; p < roff + cnt_r; ++p) {
              rem -= fs[p];
              fs[p] = rem;  // downstream sum after this pair
            }
          }
          if (MODE == kGrad) __syncthreads();
          // ---- P7: Gaussian-parallel reduction in cell order
          if ((MODE == kContrib || MODE == kGrad) && mine) {
            const int jw = tid >> 5;
            const uint32_t below = ((1u << lane) - 1u) & range_mask(jw, j0, j1);
            const uint32_t pshift = 8 * (jw & 3);
            const uint32_t* wp = wpre + (jw < 4 ? 0 : kRays);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              uint64_t m = lm[w];
              while (m) {
                const int b = __ffsll((long long)m) - 1;
                m &= m - 1;
                const int r = w * 64 + b;
                const int p = ray_off[r] + (int)((wp[r] >> pshift) & 255u) + __popc(rows[jw * kRays + r] & below);
                if (MODE == kContrib) {
                  racc[0] += fs[p];
                } else {
                  const double dx = dsub((double)(tx * kTile + (r & 15)), su[tid]);
                  const double dy = dsub((double)(ty * kTile + (r >> 4)), sv[tid]);
                  const double y2 = (fx[p] - fs[p]) * fw[p];
                  grad_terms(fy[p], y2, sk[tid], dx, dy, sa0[tid], sa1[tid], sa2[tid], racc);
                }
              }
            }
          }
        }
        __syncthreads();
        j0 = j1;
      }
      if (MODE == kContrib && have) a.partial[pos] = racc[0];
      if (MODE == kGrad && have) {
        double4* rec = reinterpret_cast<double4*>(a.partial + (int64_t)pos * 8);
        rec[0] = make_double4(racc[0] * sg[tid], racc[1], racc[2], racc[3]);
        rec[1] = make_double4(racc[4], racc[5], racc[6], 0.0);
      }
    }
    // every Gaussian of the segment owns a record: zero the ones past an early exit
    if (MODE == kContrib || MODE == kGrad) {
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
static int walk_grid(int max_items) {
  static int per_sm = 0;
  static int sms = 0;
  if (per_sm == 0) {
    const size_t smem = WalkCfg<MODE>::kSmem;
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
  if (cudaMemsetAsync(a.counter, 0, sizeof(uint32_t), st) != cudaSuccess) return SDGR_ERR_CUDA;
  const int grid = walk_grid<MODE>(max_items);
  k_walk<MODE><<<grid, 256, WalkCfg<MODE>::kSmem, st>>>(a);
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
