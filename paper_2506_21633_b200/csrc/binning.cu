// binning.cu — K2-K5: depth-rank sort, (tile, Gaussian) pair emission,
// stable tile sort, per-tile ranges and depth-segment work items.
//
// Reference: forward.build_ray_lists (forward.py:138-155) sorts every
// (cell, Gaussian) pair with np.lexsort((prim, depth, cell)); the splat pairs
// use np.lexsort((prim, pixel)) (forward.py:220).  Here the same orders are
// produced at 16x16-tile granularity:
//   1. one stable LSD radix sort of the N FP64 depth keys (+ index) -> rank
//   2. pairs emitted in rank order (comp) or index order (imaging)
//   3. one stable LSD radix sort of the pairs by tile id
// so each tile's list is ordered by (depth, index) / index, bit-exactly the
// order the reference walks each ray.
//
// The radix sort is a single-pass-per-digit "onesweep" design: one upfront
// histogram kernel for all digits, then per 8-bit digit one kernel that ranks
// its 2048-key tile with warp match-ranking, resolves its global offset by
// decoupled look-back (4 predecessors per step: with a whole 1M-key pass
// resident in one wave, a one-at-a-time look-back chain dominated -- see
// profiles/ROUND1.md), and scatters through shared memory.  A chain-free
// three-kernel pass (count / scan / scatter) was measured slower (41 vs 24 us).
#include "common.cuh"

namespace sdgr {

#ifndef SDGR_SORT_IPT
#define SDGR_SORT_IPT 8
#endif
#ifndef SDGR_SORT_MATCH
#define SDGR_SORT_MATCH 1  // MATCH.ANY measured ~4% faster than the 9-ballot split here
#endif
#ifndef SDGR_SORT_LB
#define SDGR_SORT_LB 4
#endif
constexpr int kSortThreads = 256;
constexpr int kSortIpt = SDGR_SORT_IPT;
constexpr int kLookback = SDGR_SORT_LB;  // predecessor statuses loaded per look-back step
constexpr int kSortTile = kSortThreads * kSortIpt;  // 2048
constexpr uint32_t kFlagA = 1u << 30, kFlagP = 2u << 30, kCountMask = (1u << 30) - 1;

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// ------------------------------------------------------------ histogram ----
// Item counts may live on the device (n_dev != NULL): the host passes a
// capacity n and the kernels use min(*n_dev, n), so the whole binning chain
// runs without a host round trip (and can be graph-captured).
__device__ __forceinline__ int64_t eff_count(int64_t n, const int32_t* n_dev) {
  if (!n_dev) return n;
  const int64_t d = *n_dev;
  return d < n ? d : n;
}

template <typename K>
__global__ void __launch_bounds__(256) k_radix_hist(const K* __restrict__ keys, int64_t n_cap,
                                                    const int32_t* n_dev, int begin_bit, int npass,
                                                    uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[8][256];
  const int64_t n = eff_count(n_cap, n_dev);
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const K k = keys[i];
    for (int p = 0; p < npass; ++p) atomicAdd(&sh[p][(uint32_t)(k >> (begin_bit + 8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
    const uint32_t c = (&sh[0][0])[i];
    if (c) atomicAdd(hist + i, c);
  }
}

// ------------------------------------------------------------- onesweep ----
template <typename K, bool kIota>
__global__ void __launch_bounds__(kSortThreads) k_onesweep(
    const K* __restrict__ kin, const uint32_t* __restrict__ vin, K* __restrict__ kout,
    uint32_t* __restrict__ vout, int64_t n_cap, const int32_t* n_dev, int shift,
    const uint32_t* __restrict__ ghist, uint32_t* status, uint32_t* counter) {
  const int64_t n = eff_count(n_cap, n_dev);
  extern __shared__ __align__(16) unsigned char dyn[];
  K* skeys = reinterpret_cast<K*>(dyn);
  uint32_t* svals = reinterpret_cast<uint32_t*>(dyn + sizeof(K) * kSortTile);
  __shared__ uint32_t whist[kSortThreads / 32][256];
  __shared__ uint32_t dstart[256];
  __shared__ int64_t goff[256];
  __shared__ uint32_t scan_tmp[16];
  __shared__ int bid_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) bid_s = (int)atomicAdd(counter, 1u);
  for (int i = tid; i < (kSortThreads / 32) * 256; i += kSortThreads) (&whist[0][0])[i] = 0;
  __syncthreads();
  const int bid = bid_s;
  const int64_t tile0 = (int64_t)bid * kSortTile;
  if (tile0 >= n && bid > 0) return;  // beyond the device count: nobody waits on us
  const uint32_t lt = (1u << lane) - 1u;

  K keys[kSortIpt];
  uint32_t vals[kSortIpt];
  uint32_t rank[kSortIpt];
  uint32_t dig[kSortIpt];
#pragma unroll
  for (int i = 0; i < kSortIpt; ++i) {
    const int64_t idx = tile0 + warp * (32 * kSortIpt) + i * 32 + lane;
    const bool valid = idx < n;
    keys[i] = valid ? kin[idx] : K(0);
    vals[i] = valid ? (kIota ? (uint32_t)idx : vin[idx]) : 0u;
    dig[i] = valid ? ((uint32_t)(keys[i] >> shift) & 255u) : 256u;
  }
#pragma unroll
  for (int i = 0; i < kSortIpt; ++i) {
    const uint32_t d = dig[i];
#if SDGR_SORT_MATCH
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
#else
    // warp multi-split by ballots (9 bits: 8 digit bits + the invalid flag);
    // cheaper than MATCH.ANY, which serialises on the MIO pipe
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 9; ++b) {
      const bool bit = (d >> b) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, bit);
      peers &= bit ? bal : ~bal;
    }
#endif
    uint32_t before = 0;
    if (d < 256) before = whist[warp][d];
    rank[i] = before + __popc(peers & lt);
    __syncwarp();
    if (d < 256 && lane == __ffs(peers) - 1) whist[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive offsets across warps, block total
  const int t = tid;  // digit owned by this thread
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < kSortThreads / 32; ++w) {
    const uint32_t c = whist[w][t];
    whist[w][t] = total;
    total += c;
  }
  // publish aggregate / inclusive prefix
  volatile uint32_t* vstat = status;
  if (bid == 0) vstat[t] = kFlagP | total;
  else vstat[(int64_t)bid * 256 + t] = kFlagA | total;
  // block-local exclusive scans over digits: this tile's totals, and the
  // pass's global digit histogram (-> the digit's global base offset)
  const uint32_t h = ghist[t];
  uint32_t x = total, xh = h;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
    const uint32_t yh = __shfl_up_sync(0xffffffffu, xh, off);
    if (lane >= off) { x += y; xh += yh; }
  }
  if (lane == 31) { scan_tmp[warp] = x; scan_tmp[8 + warp] = xh; }
  __syncthreads();
  uint32_t wpre = 0, wpreh = 0;
  for (int w = 0; w < warp; ++w) { wpre += scan_tmp[w]; wpreh += scan_tmp[8 + w]; }
  const uint32_t excl = wpre + x - total;
  const uint32_t gbase = wpreh + xh - h;
  dstart[t] = excl;
  // decoupled look-back for this digit
  uint32_t prefix = 0;
  if (bid > 0) {
    // 4-wide window: the four predecessor statuses are loaded together, so
    // a chain of aggregate-only blocks costs 1/4 of the dependent loads
    int64_t j = bid - 1;
    bool done = false;
    while (!done) {
      uint32_t s[kLookback];
#pragma unroll
      for (int k = 0; k < kLookback; ++k)
        s[k] = (j - k >= 0) ? (uint32_t)vstat[(j - k) * 256 + t] : (uint32_t)(2u << 30);
      int k = 0;
      for (; k < kLookback; ++k) {
        const uint32_t f = s[k] & ~kCountMask;
        if (f == 0) break;               // not published yet: retry from here
        prefix += s[k] & kCountMask;
        if (f == kFlagP) { done = true; break; }
      }
      if (!done) j -= k;
    }
    vstat[(int64_t)bid * 256 + t] = kFlagP | (prefix + total);
  }
  goff[t] = (int64_t)gbase + prefix - excl;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kSortIpt; ++i) {
    const uint32_t d = dig[i];
    if (d < 256) {
      const uint32_t lp = dstart[d] + whist[warp][d] + rank[i];
      skeys[lp] = keys[i];
      svals[lp] = vals[i];
    }
  }
  __syncthreads();
  const int64_t rem = n - tile0;
  const int cnt = rem < kSortTile ? (int)rem : kSortTile;
  for (int i = tid; i < cnt; i += kSortThreads) {
    const K k = skeys[i];
    const uint32_t d = (uint32_t)(k >> shift) & 255u;
    const int64_t gp = goff[d] + i;
    kout[gp] = k;
    vout[gp] = svals[i];
  }
}

template <typename K>
size_t radix_ws_bytes(int64_t n, int npass) {
  const int64_t nblk = (n + kSortTile - 1) / kSortTile;
  size_t b = 0;
  b += align_up(sizeof(uint32_t) * 8 * 256);                  // hist
  b += align_up(sizeof(uint32_t) * 8);                        // counters
  b += align_up(sizeof(uint32_t) * (size_t)npass * nblk * 256);  // status
  b += align_up(sizeof(K) * (size_t)n);                       // alt keys
  b += align_up(sizeof(uint32_t) * (size_t)n);                // alt vals
  return b;
}

template <typename K>
void set_sort_smem() {
  static bool done = false;
  if (done) return;
  const int bytes = (int)((sizeof(K) + 4) * kSortTile);
  cudaFuncSetAttribute(k_onesweep<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_onesweep<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done = true;
}

// Stable sort of (key, value) by key bits [begin_bit, end_bit).  vin == NULL
// means values are the input positions.  Output lands in kout/vout.
template <typename K>
int radix_sort(const K* kin, const uint32_t* vin, K* kout, uint32_t* vout, int64_t n,
               const int32_t* n_dev, int begin_bit, int end_bit, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  if (n <= 0) return SDGR_OK;
  const int npass = (end_bit - begin_bit + 7) / 8;
  if (npass < 1 || npass > 8) return SDGR_ERR_INVALID;
  if (ws_bytes < radix_ws_bytes<K>(n, npass)) return SDGR_ERR_CAPACITY;
  set_sort_smem<K>();
  const int64_t nblk = (n + kSortTile - 1) / kSortTile;
  char* p = static_cast<char*>(ws);
  uint32_t* hist = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * 8 * 256);
  uint32_t* ctr = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * 8);
  uint32_t* status = reinterpret_cast<uint32_t*>(p);
  const size_t status_bytes = sizeof(uint32_t) * (size_t)npass * nblk * 256;
  p += align_up(status_bytes);
  K* kalt = reinterpret_cast<K*>(p); p += align_up(sizeof(K) * (size_t)n);
  uint32_t* valt = reinterpret_cast<uint32_t*>(p);
  // hist, counters and status are contiguous: one memset
  if (cudaMemsetAsync(hist, 0, (size_t)((char*)status - (char*)hist) + status_bytes, st) !=
      cudaSuccess)
    return SDGR_ERR_CUDA;
  const int hist_blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 2);  // fewer global bin REDs
  k_radix_hist<K><<<hist_blocks, 256, 0, st>>>(kin, n, n_dev, begin_bit, npass, hist);
  note_launch();
  const size_t smem = (sizeof(K) + 4) * kSortTile;
  const K* ki = kin;
  const uint32_t* vi = vin;
  for (int pass = 0; pass < npass; ++pass) {
    // the last pass must land in kout: alternate so that it does
    const bool to_out = ((npass - 1 - pass) % 2) == 0;
    K* ko = to_out ? kout : kalt;
    uint32_t* vo = to_out ? vout : valt;
    uint32_t* stat = status + (size_t)pass * nblk * 256;
    {
      KernelTimer kt(SDGR_K_ONESWEEP, st);
      if (pass == 0 && vin == nullptr)
        k_onesweep<K, true><<<(unsigned)nblk, kSortThreads, smem, st>>>(
            ki, vi, ko, vo, n, n_dev, begin_bit + 8 * pass, hist + pass * 256, stat, ctr + pass);
      else
        k_onesweep<K, false><<<(unsigned)nblk, kSortThreads, smem, st>>>(
            ki, vi, ko, vo, n, n_dev, begin_bit + 8 * pass, hist + pass * 256, stat, ctr + pass);
    }
    note_launch();
    ki = ko;
    vi = vo;
  }
  return check_launch();
}

template int radix_sort<uint64_t>(const uint64_t*, const uint32_t*, uint64_t*, uint32_t*,
                                  int64_t, const int32_t*, int, int, void*, size_t, cudaStream_t);
template int radix_sort<uint32_t>(const uint32_t*, const uint32_t*, uint32_t*, uint32_t*,
                                  int64_t, const int32_t*, int, int, void*, size_t, cudaStream_t);
template size_t radix_ws_bytes<uint64_t>(int64_t, int);
template size_t radix_ws_bytes<uint32_t>(int64_t, int);

// --------------------------------------------------------------- scan ------
// --------------------------------------------------------------- scan ------
// Exclusive scan of v(i) = ntiles[order ? order[i] : i] into out[0..n],
// out[n] = total.  Three phases: tile sums, scan of sums, tile rescans.
constexpr int kScanTile = 2048;  // 256 threads x 8

struct TileCount {
  const int32_t* ntiles;
  const int32_t* order;
  __device__ __forceinline__ int32_t operator()(int64_t i) const {
    return ntiles[order ? order[i] : i];
  }
};

__device__ __forceinline__ int32_t block_excl_scan(int32_t x, int32_t* tmp, int32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t s = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, s, off);
    if (lane >= off) s += y;
  }
  if (lane == 31) tmp[warp] = s;
  __syncthreads();
  int32_t pre = 0, tot = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    if (w < warp) pre += tmp[w];
    tot += tmp[w];
  }
  __syncthreads();
  total = tot;
  return pre + s - x;
}

__global__ void __launch_bounds__(256) k_scan_reduce(TileCount f, int64_t n, int32_t* sums) {
  __shared__ int32_t tmp[8];
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
  int32_t acc = 0;
  for (int i = 0; i < 8; ++i) {
    const int64_t idx = t0 + i * 256 + threadIdx.x;
    if (idx < n) acc += f(idx);
  }
  int32_t total;
  block_excl_scan(acc, tmp, total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_sums(int32_t* sums, int64_t nb) {
  __shared__ int32_t tmp[32];
  int32_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += 1024) {
    const int64_t i = b0 + threadIdx.x;
    const int32_t v = i < nb ? sums[i] : 0;
    int32_t total;
    const int32_t e = block_excl_scan(v, tmp, total);
    if (i < nb) sums[i] = carry + e;
    carry += total;
  }
}

__global__ void __launch_bounds__(256) k_scan_down(TileCount f, int64_t n, const int32_t* sums,
                                                   int32_t* out) {
  __shared__ int32_t tmp[8];
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 8;  // blocked
  int32_t v[8];
  int32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t idx = t0 + i;
    v[i] = idx < n ? f(idx) : 0;
    acc += v[i];
  }
  int32_t total;
  int32_t run = sums[blockIdx.x] + block_excl_scan(acc, tmp, total);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t idx = t0 + i;
    if (idx < n) out[idx] = run;
    run += v[i];
    if (idx == n - 1) out[n] = run;
  }
}

size_t scan_ws_bytes(int64_t n) { return align_up(sizeof(int32_t) * ((n + kScanTile - 1) / kScanTile + 1)); }

int scan_counts(const int32_t* ntiles, const int32_t* order, int64_t n, int32_t* out, void* ws,
                cudaStream_t st) {
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  int32_t* sums = static_cast<int32_t*>(ws);
  TileCount f{ntiles, order};
  k_scan_reduce<<<(unsigned)nb, 256, 0, st>>>(f, n, sums);
  k_scan_sums<<<1, 1024, 0, st>>>(sums, nb);
  k_scan_down<<<(unsigned)nb, 256, 0, st>>>(f, n, sums, out);
  note_launch(3);
  return check_launch();
}

// --------------------------------------------------------- pair emission ----
// One thread per list position i (rank for the comp plane, index for the
// imaging plane): emit the member tiles of Gaussian g = order[i] at
// offsets[i].  Tiles come from the 8x8 tile window bitmask, or for huge
// footprints from an exact FP64 re-enumeration (same test as k_project).
__global__ void __launch_bounds__(256) k_emit_pairs(sdgr_plane pl, const int32_t* order,
                                                    const int32_t* offsets, int64_t n,
                                                    int tiles_x, double cutoff,
                                                    uint32_t* keys, int32_t* vals,
                                                    int32_t* pair_start, int64_t cap,
                                                    int32_t* overflow) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t g = order ? order[i] : (int32_t)i;
  const int32_t cnt = pl.n_tiles[g];
  int64_t o = offsets[i];
  pair_start[g] = (int32_t)o;
  if (cnt == 0) return;
  // caller's pair buffers too small: flag it and emit only the pairs that fit,
  // so every slot below the capacity still holds a real (tile, Gaussian) pair
  // and the (discarded) rest of the step stays in bounds
  if (o + cnt > cap) *overflow = 1;
  if (o >= cap) return;
  const short4 bb = reinterpret_cast<const short4*>(pl.bbox)[g];
  const int tx0 = bb.x >> 4, tx1 = bb.y >> 4, ty0 = bb.z >> 4, ty1 = bb.w >> 4;
  if ((tx1 - tx0) < 8 && (ty1 - ty0) < 8) {
    uint64_t m = pl.tile_mask[g];
    while (m) {
      const int b = __ffsll((long long)m) - 1;
      m &= m - 1;
      const int tx = tx0 + (b & 7), ty = ty0 + (b >> 3);
      keys[o] = (uint32_t)(ty * tiles_x + tx);
      vals[o] = g;
      if (++o >= cap) return;
    }
    return;
  }
  const bool dense = !isfinite(cutoff);
  const double2 uv = reinterpret_cast<const double2*>(pl.uv)[g];
  const double4 A = reinterpret_cast<const double4*>(pl.inv_cov)[g];
  const double cut2 = dmul(cutoff, cutoff), a01x2 = dmul(2.0, A.y);
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      bool hit = dense;
      const int cx0 = max((int)bb.x, tx * kTile), cx1 = min((int)bb.y, tx * kTile + kTile - 1);
      const int cy0 = max((int)bb.z, ty * kTile), cy1 = min((int)bb.w, ty * kTile + kTile - 1);
      for (int iv = cy0; iv <= cy1 && !hit; ++iv) {
        const double dy = dsub((double)iv, uv.y);
        const double t3 = dmul(A.z, dmul(dy, dy));
        for (int iu = cx0; iu <= cx1; ++iu) {
          const double dx = dsub((double)iu, uv.x);
          const double q = dadd(dadd(dmul(A.x, dmul(dx, dx)), dmul(dmul(a01x2, dx), dy)), t3);
          if (q <= cut2) { hit = true; break; }
        }
      }
      if (hit) {
        keys[o] = (uint32_t)(ty * tiles_x + tx);
        vals[o] = g;
        if (++o >= cap) return;
      }
    }
}

// scene index of each sorted pair: pair_prim[i] = pre_prim[pair_pos[i]]
// ... and, for the computation plane, the packed record the tile walks read
// coalesced instead of gathering from the N-sized projection records.
// Also the CSR tile ranges of the non-empty tiles, from the run boundaries of
// the sorted tile ids (range was preset to -1; k_make_items fills the empty
// tiles' [s, s]).
__global__ void __launch_bounds__(256) k_gather_prim(const int32_t* pos, const int32_t* pre, int64_t n_cap,
                                                     const int32_t* n_dev, int32_t* prim,
                                                     sdgr_plane pl, const double* kappa,
                                                     const double* phase, sdgr_pair_rec* rec,
                                                     const uint32_t* keys, int32_t* range) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = eff_count(n_cap, n_dev);
  if (i >= n) return;
  const uint32_t t = keys[i];
  if (i == 0 || keys[i - 1] != t) range[2 * t] = (int32_t)i;
  if (i == n - 1 || keys[i + 1] != t) range[2 * t + 1] = (int32_t)(i + 1);
  const int32_t p = pos[i];
  const int32_t g = pre[p];
  prim[i] = g;
  if (!rec) return;
  const double2 uv = reinterpret_cast<const double2*>(pl.uv)[g];
  const double4 A = reinterpret_cast<const double4*>(pl.inv_cov)[g];
  const short4 bb = reinterpret_cast<const short4*>(pl.bbox)[g];
  double4* r = reinterpret_cast<double4*>(rec + i);
  r[0] = make_double4(uv.x, uv.y, A.x, A.y);
  r[1] = make_double4(A.z, kappa[g], phase[g], __longlong_as_double((long long)pl.cell_mask[g]));
  int4 tail;
  tail.x = (int)(unsigned short)bb.x | ((int)bb.y << 16);
  tail.y = (int)(unsigned short)bb.z | ((int)bb.w << 16);
  tail.z = p;
  tail.w = g;
  reinterpret_cast<int4*>(rec + i)[4] = tail;
}

// depth-segment work items: each tile list is cut into segments of at most
// seg_len Gaussians; items are tile-major, segment-minor.
__global__ void __launch_bounds__(1024) k_make_items(int32_t* range, int n_tiles, int seg_len,
                                                     int max_items, int32_t* items,
                                                     int32_t* tile_first, int32_t* n_items,
                                                     int32_t* overflow, int64_t n_cap, const int32_t* n_dev) {
  __shared__ int32_t tmp[32];
  // empty tiles (range still -1): [s, s] with s = start of the next non-empty
  // tile, or the pair count -- a suffix min over tiles, chunks last to first
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t after = (int32_t)eff_count(n_cap, n_dev);
    const int n_chunks = (n_tiles + 1023) / 1024;
    for (int c = n_chunks - 1; c >= 0; --c) {
      const int t = c * 1024 + (1023 - (int)threadIdx.x);   // thread 0 = last tile of the chunk
      const int32_t s0 = t < n_tiles ? range[2 * t] : -1;
      int32_t m = s0 < 0 ? INT32_MAX : s0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int32_t o = __shfl_up_sync(0xffffffffu, m, off);
        if (lane >= off) m = min(m, o);
      }
      if (lane == 31) tmp[warp] = m;
      __syncthreads();
      int32_t pre = after;
      for (int w = 0; w < warp; ++w) pre = min(pre, tmp[w]);
      m = min(m, pre);
      if (t < n_tiles && s0 < 0) { range[2 * t] = m; range[2 * t + 1] = m; }
      int32_t all = after;
      for (int w = 0; w < 32; ++w) all = min(all, tmp[w]);
      __syncthreads();
      after = all;
    }
    __syncthreads();
  }
  int32_t carry = 0;
  for (int t0 = 0; t0 < n_tiles; t0 += 1024) {
    const int t = t0 + threadIdx.x;
    int32_t nseg = 0, s = 0, e = 0;
    if (t < n_tiles) {
      s = range[2 * t];
      e = range[2 * t + 1];
      nseg = (e - s + seg_len - 1) / seg_len;
    }
    int32_t total;
    const int32_t first = carry + block_excl_scan(nseg, tmp, total);
    if (t < n_tiles) {
      tile_first[t] = first;
      for (int k = 0; k < nseg; ++k) {
        const int it = first + k;
        if (it < max_items) {
          items[4 * it + 0] = t;
          items[4 * it + 1] = s + k * seg_len;
          items[4 * it + 2] = min(e, s + (k + 1) * seg_len);
          items[4 * it + 3] = first;
        }
      }
    }
    carry += total;
  }
  if (threadIdx.x == 0) {
    *n_items = carry < max_items ? carry : max_items;
    if (carry > max_items) *overflow = 1;
  }
}

int launch_emit_and_sort(const sdgr_projection& proj, const sdgr_view& view, const int32_t* order,
                         const int32_t* offsets, sdgr_tiles& tl, void* ws, size_t ws_bytes,
                         cudaStream_t st) {
  const sdgr_plane& pl = tl.plane == 0 ? proj.comp : proj.img;
  const int64_t n = proj.n, np = tl.n_pairs;  // np: exact count, or capacity with a device count
  // device-side pair count = offsets[n] (the scan's total) when capacity mode is on
  const int32_t* n_dev = tl.device_count ? offsets + n : nullptr;
  if (cudaMemsetAsync(tl.tile_range, 0xff, sizeof(int32_t) * 2 * (size_t)tl.n_tiles, st) != cudaSuccess)
    return SDGR_ERR_CUDA;
  // n_items[0] is written by k_make_items; n_items[1] (overflow) is sticky
  // until the caller clears it, so one check can cover many views.
  int32_t* overflow = tl.n_items + 1;
  if (np > 0) {
    char* p = static_cast<char*>(ws);
    uint32_t* keys = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * np);
    const size_t used = (size_t)(p - static_cast<char*>(ws));
    if (used > ws_bytes) return SDGR_ERR_CAPACITY;
    {
      KernelTimer kt(SDGR_K_EMIT, st);
      k_emit_pairs<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pl, order, offsets, n, tl.tiles_x,
                                                                view.cutoff, keys, tl.pre_prim,
                                                                tl.pair_start, np, overflow);
    }
    note_launch();
    int bits = 1;
    while ((1 << bits) < tl.n_tiles) ++bits;
    // stable by tile; values = pre-sort positions (iota)
    const int rc = radix_sort<uint32_t>(keys, nullptr, tl.pair_tile,
                                        reinterpret_cast<uint32_t*>(tl.pair_pos), np, n_dev, 0, bits,
                                        p, ws_bytes - used, st);
    if (rc != SDGR_OK) return rc;
    {
      KernelTimer kt(SDGR_K_GATHER, st);
      k_gather_prim<<<(unsigned)((np + 255) / 256), 256, 0, st>>>(tl.pair_pos, tl.pre_prim, np, n_dev,
                                                                  tl.pair_prim, pl, proj.kappa, proj.phase,
                                                                  tl.plane == 0 ? tl.pair_rec : nullptr,
                                                                  tl.pair_tile, tl.tile_range);
    }
    note_launch();
  } else {
    k_emit_pairs<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pl, order, offsets, n, tl.tiles_x,
                                                              view.cutoff, nullptr, nullptr,
                                                              tl.pair_start, 0, overflow);
    note_launch();
  }
  k_make_items<<<1, 1024, 0, st>>>(tl.tile_range, tl.n_tiles, tl.seg_len, tl.max_items, tl.items,
                                   tl.tile_first, tl.n_items, overflow, np, n_dev);
  note_launch();
  return check_launch();
}

size_t binning_ws_bytes(int64_t n, int64_t max_pairs) {
  // depth sort: range + 32-bit keys (2 arrays) + radix scratch (4 passes of 32-bit keys)
  const size_t depth = align_up(16) + 2 * align_up(sizeof(uint32_t) * (size_t)n) +
                       radix_ws_bytes<uint32_t>(n, 4);
  // pair sort: keys + radix scratch (up to 2 passes of 32-bit keys)
  const size_t pairs = align_up(sizeof(uint32_t) * (size_t)max_pairs) +
                       radix_ws_bytes<uint32_t>(max_pairs, 2);
  const size_t scan = scan_ws_bytes(n);
  return std::max(std::max(depth, pairs), scan) + 4096;
}

// ------------------------------------------------------ depth order --------
// Exact stable (FP64 depth, index) order with a 24-bit radix sort:
//   1. min / max of the visible depth keys;
//   2. k = floor((d - dmin) * (2^24 - 2) / (dmax - dmin)): monotone
//      non-decreasing in d (every FP64 step is monotone), invisible = 2^24 - 1;
//   3. stable 3-pass radix sort of k (ties keep index order);
//   4. runs of equal k (depths closer than (dmax-dmin)/2^24; ~1.3 keys per
//      run on c4) are re-sorted by the full 64-bit key, index as tie-break --
//      exactly np.lexsort's (depth, index) order (forward.py:147), with 3
//      passes instead of the 8 of a 64-bit sort.
constexpr int kKeyBits = 24;
constexpr uint32_t kKeyInvisible = (1u << kKeyBits) - 1u;
constexpr uint32_t kKeyMax = kKeyInvisible - 1u;

__device__ __forceinline__ double key_to_depth(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void __launch_bounds__(256) k_key_range(const uint64_t* key, int64_t n, unsigned long long* range) {
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = key[i];
    if (k != ~0ull) {
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const unsigned long long a = __shfl_down_sync(0xffffffffu, lo, off);
    const unsigned long long b = __shfl_down_sync(0xffffffffu, hi, off);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  // one RED pair per block: same-address atomics serialise at L2
  __shared__ unsigned long long s_lo[8], s_hi[8];
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s_lo[warp] = lo; s_hi[warp] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = s_lo[w] < lo ? s_lo[w] : lo;
      hi = s_hi[w] > hi ? s_hi[w] : hi;
    }
    atomicMin(range, lo);
    atomicMax(range + 1, hi);
  }
}

__global__ void __launch_bounds__(256) k_key32(const uint64_t* key, int64_t n, const unsigned long long* range,
                                               uint32_t* k32) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = key[i];
  if (k == ~0ull) { k32[i] = kKeyInvisible; return; }
  const double dmin = key_to_depth(range[0]), dmax = key_to_depth(range[1]);
  const double span = dsub(dmax, dmin);
  double q = 0.0;
  if (span > 0.0) q = dmul(dsub(key_to_depth(k), dmin), (double)kKeyMax / span);
  k32[i] = (uint32_t)fmin(fmax(q, 0.0), (double)kKeyMax);
}

// one thread per run of equal k32 (runs are rare and short); stable by index
__global__ void __launch_bounds__(256) k_fix_runs(const uint32_t* k32s, const uint64_t* key, int64_t n,
                                                  int32_t* order) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t k = k32s[i];
  if (k == kKeyInvisible) return;                     // invisible tail: order irrelevant
  if (i > 0 && k32s[i - 1] == k) return;               // not a run start
  if (i + 1 >= n || k32s[i + 1] != k) return;          // run of length 1
  int64_t e = i + 1;
  while (e < n && k32s[e] == k) ++e;
  for (int64_t a = i + 1; a < e; ++a) {                // insertion sort by (key, index)
    const int32_t g = order[a];
    const uint64_t kg = key[g];
    int64_t b = a - 1;
    while (b >= i) {
      const int32_t h = order[b];
      const uint64_t kh = key[h];
      if (kh < kg || (kh == kg && h < g)) break;
      order[b + 1] = h;
      --b;
    }
    order[b + 1] = g;
  }
}

int launch_depth_order(const sdgr_projection& proj, int32_t* order, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
  const int64_t n = proj.n;
  char* p = static_cast<char*>(ws);
  unsigned long long* range = reinterpret_cast<unsigned long long*>(p); p += align_up(16);
  uint32_t* k32 = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * (size_t)n);
  uint32_t* k32s = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * (size_t)n);
  const size_t used = (size_t)(p - static_cast<char*>(ws));
  if (used > ws_bytes) return SDGR_ERR_CAPACITY;
  if (cudaMemsetAsync(range, 0xff, sizeof(unsigned long long), st) != cudaSuccess ||
      cudaMemsetAsync(range + 1, 0, sizeof(unsigned long long), st) != cudaSuccess)
    return SDGR_ERR_CUDA;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  k_key_range<<<std::min<unsigned>(blocks, 148 * 2), 256, 0, st>>>(proj.depth_key, n, range);
  k_key32<<<blocks, 256, 0, st>>>(proj.depth_key, n, range, k32);
  note_launch(2);
  const int rc = radix_sort<uint32_t>(k32, nullptr, k32s, reinterpret_cast<uint32_t*>(order), n, nullptr, 0,
                                      kKeyBits, p, ws_bytes - used, st);
  if (rc != SDGR_OK) return rc;
  k_fix_runs<<<blocks, 256, 0, st>>>(k32s, proj.depth_key, n, order);
  note_launch();
  return check_launch();
}

}  // namespace sdgr
