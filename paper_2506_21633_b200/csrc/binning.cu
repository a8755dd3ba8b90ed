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
// Every stage is batched over up to SDGR_MAX_BATCH views of one scene: one
// launch covers all views (per-view pointers travel in the kernel parameter
// block, the view is blockIdx.y or part of the flattened block id).  A 1M-key
// sort or a 1M-entry scan is far too small to fill 148 SMs on its own -- the
// single-view passes were look-back- and launch-latency bound (profiles/) --
// so batching the views is what turns these stages bandwidth-shaped.  The
// single-view entry points are batches of one.
//
// The radix sort is a single-pass-per-digit "onesweep" design: the digit
// histograms come from the kernel that produces the keys (fused), then per
// 8-bit digit one kernel ranks its 2048-key tile with warp match-ranking,
// resolves its global offset by decoupled look-back (4 predecessors per step)
// and scatters through shared memory.  Blocks take their (view, tile) from
// one atomic ticket, views interleaved, so each view's look-back chain only
// ever waits on blocks that already started.
#include "common.cuh"

namespace sdgr {

#ifndef SDGR_SORT_IPT
#define SDGR_SORT_IPT 16   // 16 keys per thread: the 5 sort passes 1.91 -> 1.84 ms/step (8: round 1)
#endif
#ifndef SDGR_SORT_MATCH
#define SDGR_SORT_MATCH 0  // 9-ballot split: 5% faster than MATCH.ANY once the passes were batched
#endif
#ifndef SDGR_SORT_LB
#define SDGR_SORT_LB 4
#endif
#ifndef SDGR_SORT_MINB
#define SDGR_SORT_MINB 3   // resident blocks per SM (register cap 80; 4: 64 with spills, passes 1.843 vs 1.831 ms/step)
#endif
constexpr int kMaxBatch = SDGR_MAX_BATCH;
constexpr int kSortThreads = 256;
constexpr int kSortIpt = SDGR_SORT_IPT;
constexpr int kLookback = SDGR_SORT_LB;  // predecessor statuses loaded per look-back step
constexpr int kSortTile = kSortThreads * kSortIpt;  // 4096
constexpr int kMaxPass = 3;                          // 24-bit keys at most (depth keys, <= 16M tiles)
constexpr int kHistStride = kMaxPass * 256;          // per-view digit histogram words
constexpr uint32_t kFlagA = 1u << 30, kFlagP = 2u << 30, kCountMask = (1u << 30) - 1;

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Item counts may live on the device (n_dev != NULL): the host passes a
// capacity n and the kernels use min(*n_dev, n), so the whole binning chain
// runs without a host round trip (and can be graph-captured).
__device__ __forceinline__ int64_t eff_count(int64_t n, const int32_t* n_dev) {
  if (!n_dev) return n;
  const int64_t d = *n_dev;
  return d < n ? d : n;
}

// blocks per view for grid-stride kernels that flush a block histogram:
// ~2 blocks per SM over the whole batch
static unsigned stride_blocks(int64_t n, int nv, int per_sm = 2) {
  const int64_t want = std::max<int64_t>(1, (int64_t)sm_count() * per_sm / nv);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, want));
}

// ------------------------------------------------------------- onesweep ----
// Per-view key / value arrays of one pass.
struct SortIO {
  const uint32_t* kin[kMaxBatch];
  const uint32_t* vin[kMaxBatch];   // unused when the pass is an iota pass
  uint32_t* kout[kMaxBatch];
  uint32_t* vout[kMaxBatch];
  const int32_t* n_dev[kMaxBatch];  // device counts (NULL: n_cap)
};

template <bool kIota>
__global__ void __launch_bounds__(kSortThreads, SDGR_SORT_MINB) k_onesweep(
    const __grid_constant__ SortIO io, int nv, int64_t n_cap, int64_t nblk, int shift, int pass,
    const uint32_t* __restrict__ ghist_all, uint32_t* status_all, uint32_t* counter) {
  extern __shared__ __align__(16) unsigned char dyn[];
  uint32_t* skeys = reinterpret_cast<uint32_t*>(dyn);
  uint32_t* svals = reinterpret_cast<uint32_t*>(dyn + sizeof(uint32_t) * kSortTile);
  __shared__ uint32_t whist[kSortThreads / 32][256];
  __shared__ uint32_t dstart[256];
  __shared__ int64_t goff[256];
  __shared__ uint32_t scan_tmp[16];
  __shared__ int bid_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) bid_s = (int)atomicAdd(counter, 1u);
  for (int i = tid; i < (kSortThreads / 32) * 256; i += kSortThreads) (&whist[0][0])[i] = 0;
  __syncthreads();
  const int view = bid_s % nv;
  const int bid = bid_s / nv;
  const int64_t n = eff_count(n_cap, io.n_dev[view]);
  const int64_t tile0 = (int64_t)bid * kSortTile;
  if (tile0 >= n && bid > 0) return;  // beyond the device count: nobody waits on us
  const uint32_t* __restrict__ kin = io.kin[view];
  const uint32_t* __restrict__ vin = io.vin[view];
  uint32_t* __restrict__ kout = io.kout[view];
  uint32_t* __restrict__ vout = io.vout[view];
  const uint32_t* ghist = ghist_all + (size_t)view * kHistStride + pass * 256;
  uint32_t* status = status_all + (size_t)view * nblk * 256;
  const uint32_t lt = (1u << lane) - 1u;

  uint32_t keys[kSortIpt];
  uint32_t vals[kSortIpt];
  uint32_t rank[kSortIpt];
  uint32_t dig[kSortIpt];
#pragma unroll
  for (int i = 0; i < kSortIpt; ++i) {
    const int64_t idx = tile0 + warp * (32 * kSortIpt) + i * 32 + lane;
    const bool valid = idx < n;
    keys[i] = valid ? kin[idx] : 0u;
    vals[i] = valid ? (kIota ? (uint32_t)idx : vin[idx]) : 0u;
    dig[i] = valid ? ((keys[i] >> shift) & 255u) : 256u;
  }
#pragma unroll
  for (int i = 0; i < kSortIpt; ++i) {
    const uint32_t d = dig[i];
#if SDGR_SORT_MATCH
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
#else
    // warp multi-split by ballots (9 bits: 8 digit bits + the invalid flag)
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
    const uint32_t k = skeys[i];
    const uint32_t d = (k >> shift) & 255u;
    const int64_t gp = goff[d] + i;
    kout[gp] = k;
    vout[gp] = svals[i];
  }
}

// Radix scratch of a batch: digit histograms (filled by the key producer),
// per-pass tickets, look-back status words, and the ping-pong key / value
// arrays (view-strided).
struct RadixWs {
  uint32_t* hist;    // [nv][kMaxPass][256]
  uint32_t* ctr;     // [kMaxPass]
  uint32_t* status;  // [kMaxPass][nv][nblk][256]
  uint32_t* kalt;    // [nv][n]
  uint32_t* valt;    // [nv][n]
  int64_t nblk;
  size_t zero_bytes; // hist .. end of status (one memset)
};

static size_t radix_ws_bytes(int64_t n, int nv) {
  const int64_t nblk = (n + kSortTile - 1) / kSortTile;
  size_t b = 0;
  b += align_up(sizeof(uint32_t) * (size_t)nv * kHistStride);
  b += align_up(sizeof(uint32_t) * kMaxPass);
  b += align_up(sizeof(uint32_t) * (size_t)kMaxPass * nv * nblk * 256);
  b += 2 * align_up(sizeof(uint32_t) * (size_t)nv * n);
  return b;
}

static RadixWs radix_layout(char*& p, int64_t n, int nv) {
  RadixWs r;
  r.nblk = (n + kSortTile - 1) / kSortTile;
  char* base = p;
  r.hist = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * (size_t)nv * kHistStride);
  r.ctr = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * kMaxPass);
  r.status = reinterpret_cast<uint32_t*>(p);
  p += align_up(sizeof(uint32_t) * (size_t)kMaxPass * nv * r.nblk * 256);
  r.zero_bytes = (size_t)(p - base);
  r.kalt = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * (size_t)nv * n);
  r.valt = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * (size_t)nv * n);
  return r;
}

static void set_sort_smem() {
  static bool done = false;
  if (done) return;
  const int bytes = (int)(8 * kSortTile);
  cudaFuncSetAttribute(k_onesweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  cudaFuncSetAttribute(k_onesweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done = true;
}

// Stable sort of each view's (key, value) by key bits [0, 8*npass), values =
// input positions (iota) when `iota`.  The digit histograms must already be
// in r.hist and the tickets / status words zeroed.  Output lands in
// io.kout / io.vout.
static int radix_passes(const SortIO& io, bool iota, int nv, int64_t n_cap, int npass, const RadixWs& r,
                        cudaStream_t st) {
  if (npass < 1 || npass > kMaxPass) return SDGR_ERR_INVALID;
  set_sort_smem();
  const size_t smem = 8 * kSortTile;
  SortIO cur = io;
  for (int pass = 0; pass < npass; ++pass) {
    // the last pass must land in kout: alternate so that it does
    const bool to_out = ((npass - 1 - pass) % 2) == 0;
    for (int v = 0; v < nv; ++v) {
      cur.kout[v] = to_out ? io.kout[v] : r.kalt + (size_t)v * n_cap;
      cur.vout[v] = to_out ? io.vout[v] : r.valt + (size_t)v * n_cap;
    }
    uint32_t* stat = r.status + (size_t)pass * nv * r.nblk * 256;
    const unsigned grid = (unsigned)(r.nblk * nv);
    {
      KernelTimer kt(SDGR_K_ONESWEEP, st);
      if (pass == 0 && iota)
        k_onesweep<true><<<grid, kSortThreads, smem, st>>>(cur, nv, n_cap, r.nblk, 8 * pass, pass, r.hist, stat,
                                                           r.ctr + pass);
      else
        k_onesweep<false><<<grid, kSortThreads, smem, st>>>(cur, nv, n_cap, r.nblk, 8 * pass, pass, r.hist, stat,
                                                            r.ctr + pass);
    }
    note_launch();
    for (int v = 0; v < nv; ++v) {
      cur.kin[v] = cur.kout[v];
      cur.vin[v] = cur.vout[v];
    }
  }
  return check_launch();
}

// block histogram of up to kMaxPass 8-bit digits, flushed to the view's slot
struct BlockHist {
  uint32_t (*sh)[256];
  __device__ void clear() {
    for (int i = threadIdx.x; i < kMaxPass * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
  }
  __device__ void add(uint32_t k, int npass) {
    for (int p = 0; p < npass; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 255u], 1u);
  }
  __device__ void flush(uint32_t* dst, int npass) {
    for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
      const uint32_t c = (&sh[0][0])[i];
      if (c) atomicAdd(dst + i, c);
    }
  }
};

// --------------------------------------------------------------- scan ------
// Exclusive scan of v(i) = ntiles[order ? order[i] : i] into out[0..n],
// out[n] = total, per view.  Three phases: tile sums, scan of sums, rescans.
constexpr int kScanTile = 2048;  // 256 threads x 8

struct ScanIO {
  const int32_t* ntiles[kMaxBatch];
  const int32_t* order[kMaxBatch];
  int32_t* out[kMaxBatch];
};

__device__ __forceinline__ int32_t tile_count(const ScanIO& io, int v, int64_t i) {
  const int32_t* o = io.order[v];
  return io.ntiles[v][o ? o[i] : i];
}

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

__global__ void __launch_bounds__(256) k_scan_reduce(const __grid_constant__ ScanIO io, int64_t n, int32_t* sums,
                                                     int64_t nb) {
  __shared__ int32_t tmp[8];
  const int v = blockIdx.y;
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
  int32_t acc = 0;
  for (int i = 0; i < 8; ++i) {
    const int64_t idx = t0 + i * 256 + threadIdx.x;
    if (idx < n) acc += tile_count(io, v, idx);
  }
  int32_t total;
  block_excl_scan(acc, tmp, total);
  if (threadIdx.x == 0) sums[v * nb + blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) k_scan_sums(int32_t* sums_all, int64_t nb) {
  __shared__ int32_t tmp[32];
  int32_t* sums = sums_all + blockIdx.x * nb;
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

__global__ void __launch_bounds__(256) k_scan_down(const __grid_constant__ ScanIO io, int64_t n,
                                                   const int32_t* sums, int64_t nb) {
  __shared__ int32_t tmp[8];
  const int vw = blockIdx.y;
  int32_t* out = io.out[vw];
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 8;  // blocked
  int32_t v[8];
  int32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t idx = t0 + i;
    v[i] = idx < n ? tile_count(io, vw, idx) : 0;
    acc += v[i];
  }
  int32_t total;
  int32_t run = sums[vw * nb + blockIdx.x] + block_excl_scan(acc, tmp, total);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t idx = t0 + i;
    if (idx < n) out[idx] = run;
    run += v[i];
    if (idx == n - 1) out[n] = run;
  }
}

static size_t scan_ws_bytes(int64_t n, int nv) {
  return align_up(sizeof(int32_t) * (size_t)nv * ((n + kScanTile - 1) / kScanTile + 1));
}

static int scan_counts_batch(const ScanIO& io, int nv, int64_t n, void* ws, cudaStream_t st) {
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  int32_t* sums = static_cast<int32_t*>(ws);
  k_scan_reduce<<<dim3((unsigned)nb, nv), 256, 0, st>>>(io, n, sums, nb);
  k_scan_sums<<<nv, 1024, 0, st>>>(sums, nb);
  k_scan_down<<<dim3((unsigned)nb, nv), 256, 0, st>>>(io, n, sums, nb);
  note_launch(3);
  return check_launch();
}

// --------------------------------------------------------- pair emission ----
// Grid-stride over list positions i (rank for the comp plane, index for the
// imaging plane): emit the member tiles of Gaussian g = order[i] at
// offsets[i].  Tiles come from the 8x8 tile window bitmask, or for huge
// footprints from an exact FP64 re-enumeration (same test as k_project).
// The tile sort's digit histograms are accumulated on the way.
struct EmitIO {
  sdgr_plane pl[kMaxBatch];
  const int32_t* order[kMaxBatch];
  const int32_t* offsets[kMaxBatch];
  uint32_t* keys[kMaxBatch];
  int32_t* vals[kMaxBatch];
  int32_t* pair_start[kMaxBatch];
  int32_t* overflow[kMaxBatch];
};

__global__ void __launch_bounds__(256) k_emit_pairs(const __grid_constant__ EmitIO io, int64_t n, int tiles_x,
                                                    double cutoff, int64_t cap, uint32_t* hist, int npass) {
  __shared__ uint32_t sh[kMaxPass][256];
  BlockHist bh{sh};
  if (hist) {
    bh.clear();
    __syncthreads();
  }
  const int v = blockIdx.y;
  const sdgr_plane& pl = io.pl[v];
  const int32_t* order = io.order[v];
  uint32_t* keys = io.keys[v];
  int32_t* vals = io.vals[v];
  const bool dense = !isfinite(cutoff);
  const double cut2 = dmul(cutoff, cutoff);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = order ? order[i] : (int32_t)i;
    const int32_t cnt = pl.n_tiles[g];
    int64_t o = io.offsets[v][i];
    io.pair_start[v][g] = (int32_t)o;
    if (cnt == 0) continue;
    // caller's pair buffers too small: flag it and emit only the pairs that fit,
    // so every slot below the capacity still holds a real (tile, Gaussian) pair
    // and the (discarded) rest of the step stays in bounds
    if (o + cnt > cap) *io.overflow[v] = 1;
    if (o >= cap || !keys) continue;
    const short4 bb = reinterpret_cast<const short4*>(pl.bbox)[g];
    const int tx0 = bb.x >> 4, tx1 = bb.y >> 4, ty0 = bb.z >> 4, ty1 = bb.w >> 4;
    if ((tx1 - tx0) < 8 && (ty1 - ty0) < 8) {
      uint64_t m = pl.tile_mask[g];
      while (m && o < cap) {
        const int b = __ffsll((long long)m) - 1;
        m &= m - 1;
        const uint32_t t = (uint32_t)((ty0 + (b >> 3)) * tiles_x + tx0 + (b & 7));
        keys[o] = t;
        vals[o] = g;
        ++o;
        if (hist) bh.add(t, npass);
      }
      continue;
    }
    const double2 uv = reinterpret_cast<const double2*>(pl.uv)[g];
    const double4 A = reinterpret_cast<const double4*>(pl.inv_cov)[g];
    const double a01x2 = dmul(2.0, A.y);
    for (int ty = ty0; ty <= ty1 && o < cap; ++ty)
      for (int tx = tx0; tx <= tx1 && o < cap; ++tx) {
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
          const uint32_t t = (uint32_t)(ty * tiles_x + tx);
          keys[o] = t;
          vals[o] = g;
          ++o;
          if (hist) bh.add(t, npass);
        }
      }
  }
  if (hist) {
    __syncthreads();
    bh.flush(hist + (size_t)v * kHistStride, npass);
  }
}

// Fused count + emit (the batched multi-view path): one pass over the list
// positions does what k_scan_reduce / k_scan_sums / k_scan_down + k_emit_pairs
// do, reading each Gaussian's 16-byte emit row (bbox | tile_mask,
// sdgr_plane.emit) once.  Block = 2048 consecutive list positions; its pair
// offset comes from a single-value decoupled look-back (warp-wide window) over
// the view's earlier blocks, blocks ticketed like the onesweep passes.
#ifndef SDGR_EMIT_IPT
#define SDGR_EMIT_IPT 4
#endif
constexpr int kEmitIpt = SDGR_EMIT_IPT;
constexpr int kEmitTile = 256 * kEmitIpt;
constexpr unsigned long long kSFlagA = 1ull << 62, kSFlagP = 2ull << 62, kSValue = (1ull << 62) - 1;

struct FusedEmitIO {
  const ulonglong2* erow[kMaxBatch];
  const int32_t* ntiles[kMaxBatch];
  const double* uv[kMaxBatch];      // centre of Gaussian g at uv[uv_stride * g]
  const double* inv_cov[kMaxBatch];
  const int32_t* order[kMaxBatch];
  int32_t* offsets[kMaxBatch];
  int uv_stride[kMaxBatch];         // 2: SoA uv, 8: packed rows
  uint32_t* keys[kMaxBatch];
  int32_t* vals[kMaxBatch];
  int32_t* pair_start[kMaxBatch];
  int32_t* overflow[kMaxBatch];
};

#ifndef SDGR_EMIT_MINB
#define SDGR_EMIT_MINB 4   // 64 registers (a few spills): k_count_emit 0.876 -> 0.848 ms/step
#endif
__global__ void __launch_bounds__(256, SDGR_EMIT_MINB) k_count_emit(const __grid_constant__ FusedEmitIO io, int nv, int64_t n,
                                                    int64_t nblk, int tiles_x, double cutoff, int64_t cap,
                                                    uint32_t* hist, int npass, unsigned long long* status_all,
                                                    uint32_t* ticket) {
  __shared__ uint32_t sh[kMaxPass][256];
  __shared__ int32_t scnt[kEmitTile];
  __shared__ int32_t wtmp[8];
  __shared__ int bid_s;
  __shared__ long long base_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  BlockHist bh{sh};
  bh.clear();
  if (tid == 0) bid_s = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int v = bid_s % nv;
  const int64_t bid = bid_s / nv;
  const int64_t tile0 = bid * kEmitTile;
  const int32_t* order = io.order[v];
  const ulonglong2* erow = io.erow[v];
  int32_t g[kEmitIpt], cnt[kEmitIpt];
  ulonglong2 row[kEmitIpt];
#pragma unroll
  for (int k = 0; k < kEmitIpt; ++k) {
    const int64_t r = tile0 + k * 256 + tid;
    g[k] = r < n ? (order ? order[r] : (int32_t)r) : -1;
  }
#pragma unroll
  for (int k = 0; k < kEmitIpt; ++k) row[k] = g[k] >= 0 ? erow[g[k]] : make_ulonglong2(0x0000000100000001ull, 0ull);
#pragma unroll
  for (int k = 0; k < kEmitIpt; ++k) {
    const short4 bb = *reinterpret_cast<const short4*>(&row[k].x);
    const bool tsmall = ((bb.y >> 4) - (bb.x >> 4)) < 8 && ((bb.w >> 4) - (bb.z >> 4)) < 8;
    cnt[k] = bb.x > bb.y ? 0 : (tsmall ? __popcll(row[k].y) : io.ntiles[v][g[k]]);
    scnt[k * 256 + tid] = cnt[k];
  }
  __syncthreads();
  // exclusive scan over the tile in list order: thread t owns 8 consecutive slots
  int32_t loc[kEmitIpt], sum = 0;
#pragma unroll
  for (int j = 0; j < kEmitIpt; ++j) {
    loc[j] = sum;
    sum += scnt[tid * kEmitIpt + j];
  }
  int32_t total;
  const int32_t texcl = block_excl_scan(sum, wtmp, total);
#pragma unroll
  for (int j = 0; j < kEmitIpt; ++j) scnt[tid * kEmitIpt + j] = texcl + loc[j];
  // tile prefix: decoupled look-back over the view's earlier tiles
  if (warp == 0) {
    volatile unsigned long long* status = status_all + (size_t)v * nblk;
    unsigned long long prefix = 0;
    if (bid == 0) {
      if (lane == 0) status[0] = kSFlagP | (unsigned long long)total;
    } else {
      if (lane == 0) status[bid] = kSFlagA | (unsigned long long)total;
      int64_t j = bid - 1;
      while (true) {
        const int64_t idx = j - lane;
        const unsigned long long s = idx >= 0 ? (unsigned long long)status[idx] : (unsigned long long)(2ull << 62);
        const unsigned long long f = s & ~kSValue;
        const uint32_t pm = __ballot_sync(0xffffffffu, f == kSFlagP);
        const uint32_t nr = __ballot_sync(0xffffffffu, f == 0);
        const int fp = pm ? __ffs(pm) - 1 : 31;            // nearest inclusive prefix (or the window end)
        const uint32_t upto = fp == 31 ? 0xffffffffu : ((2u << fp) - 1u);
        if (nr & upto) continue;                           // a nearer tile has not published yet
        unsigned long long val = lane <= fp ? (s & kSValue) : 0ull;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) val += __shfl_down_sync(0xffffffffu, val, off);
        prefix += __shfl_sync(0xffffffffu, val, 0);
        if (pm) break;
        j -= 32;
      }
      if (lane == 0) status[bid] = kSFlagP | (prefix + (unsigned long long)total);
    }
    if (lane == 0) base_s = (long long)prefix;
  }
  __syncthreads();
  const int64_t base = base_s;
  if (tid == 0 && tile0 + kEmitTile >= n) io.offsets[v][n] = (int32_t)(base + total);  // T16 (device count)
  uint32_t* keys = io.keys[v];
  int32_t* vals = io.vals[v];
  const bool dense = !isfinite(cutoff);
  const double cut2 = dmul(cutoff, cutoff);
#pragma unroll
  for (int k = 0; k < kEmitIpt; ++k) {
    const int64_t r = tile0 + k * 256 + tid;
    if (r >= n) break;
    int64_t o = base + scnt[k * 256 + tid];
    io.offsets[v][r] = (int32_t)o;
    io.pair_start[v][g[k]] = (int32_t)o;
    const int32_t c = cnt[k];
    if (c == 0) continue;
    if (o + c > cap) *io.overflow[v] = 1;
    if (o >= cap || !keys) continue;
    const short4 bb = *reinterpret_cast<const short4*>(&row[k].x);
    const int tx0 = bb.x >> 4, tx1 = bb.y >> 4, ty0 = bb.z >> 4, ty1 = bb.w >> 4;
    if ((tx1 - tx0) < 8 && (ty1 - ty0) < 8) {
      uint64_t m = row[k].y;
      while (m && o < cap) {
        const int b = __ffsll((long long)m) - 1;
        m &= m - 1;
        const uint32_t t = (uint32_t)((ty0 + (b >> 3)) * tiles_x + tx0 + (b & 7));
        keys[o] = t;
        vals[o] = g[k];
        ++o;
        if (hist) bh.add(t, npass);
      }
      continue;
    }
    const double2 uv = *reinterpret_cast<const double2*>(io.uv[v] + (int64_t)io.uv_stride[v] * g[k]);
    const double4 A = reinterpret_cast<const double4*>(io.inv_cov[v])[g[k]];
    const double a01x2 = dmul(2.0, A.y);
    for (int ty = ty0; ty <= ty1 && o < cap; ++ty)
      for (int tx = tx0; tx <= tx1 && o < cap; ++tx) {
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
          const uint32_t t = (uint32_t)(ty * tiles_x + tx);
          keys[o] = t;
          vals[o] = g[k];
          ++o;
          if (hist) bh.add(t, npass);
        }
      }
  }
  if (hist) {
    __syncthreads();
    bh.flush(hist + (size_t)v * kHistStride, npass);
  }
}

// scene index of each sorted pair: pair_prim[i] = pre_prim[pair_pos[i]]
// ... and, for the computation plane, the packed record the tile walks read
// coalesced instead of gathering from the N-sized projection records.
// Also the CSR tile ranges of the non-empty tiles, from the run boundaries of
// the sorted tile ids (range was preset to -1; k_make_items fills the empty
// tiles' [s, s]).
struct GatherIO {
  const int32_t* pos[kMaxBatch];
  const int32_t* pre[kMaxBatch];
  const int32_t* n_dev[kMaxBatch];
  int32_t* prim[kMaxBatch];
  const double* uv[kMaxBatch];
  const double* inv_cov[kMaxBatch];
  const int16_t* bbox[kMaxBatch];
  const uint64_t* cell_mask[kMaxBatch];
  const double* kappa[kMaxBatch];
  const double* phase[kMaxBatch];
  const double* packed[kMaxBatch];
  const ulonglong2* erow[kMaxBatch];  // bbox source when the SoA bbox is absent
  sdgr_pair_rec* rec[kMaxBatch];
  const uint32_t* keys[kMaxBatch];
  int32_t* range[kMaxBatch];
  int32_t* n_items[kMaxBatch];   // [1]: overflow / invalid flag
  int32_t n_tiles[kMaxBatch];
};

// One thread per sorted pair.  With the computation plane's packed 64-byte
// per-Gaussian rows (sdgr_plane.packed) a pair's record is 2 sectors + the
// bbox instead of 6 scattered SoA sectors.
__global__ void __launch_bounds__(256) k_gather_prim(const __grid_constant__ GatherIO io, int64_t n_cap) {
  const int v = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = eff_count(n_cap, io.n_dev[v]);
  if ((int64_t)blockIdx.x * blockDim.x >= n) return;   // whole block beyond the count
  const bool live = i < n;
  const int64_t ii = live ? i : n - 1;                   // dead lanes redo the last pair, store nothing
  const uint32_t* keys = io.keys[v];
  int32_t* range = io.range[v];
  const uint32_t t = keys[ii];
  if (live) {
    if (t < (uint32_t)io.n_tiles[v]) {
      if (i == 0 || keys[i - 1] != t) range[2 * t] = (int32_t)i;
      if (i == n - 1 || keys[i + 1] != t) range[2 * t + 1] = (int32_t)(i + 1);
    } else {
      io.n_items[v][1] = 1;   // a tile id past the grid (a view whose ray grid is not the lists'): flagged, never written
    }
  }
  const int32_t p = io.pos[v][ii];
  const int32_t g = io.pre[v][p];
  if (live) io.prim[v][i] = g;
  sdgr_pair_rec* rec = io.rec[v];
  if (!rec) return;
  const short4 bb = io.bbox[v] ? reinterpret_cast<const short4*>(io.bbox[v])[g]
                               : *reinterpret_cast<const short4*>(&io.erow[v][g].x);
  double4 r0, r1;
  if (io.packed[v]) {
    const double4* pk = reinterpret_cast<const double4*>(io.packed[v]) + 2 * g;
    r0 = pk[0];
    r1 = pk[1];
  } else {
    const double2 uv = reinterpret_cast<const double2*>(io.uv[v])[g];
    const double4 A = reinterpret_cast<const double4*>(io.inv_cov[v])[g];
    r0 = make_double4(uv.x, uv.y, A.x, A.y);
    r1 = make_double4(A.z, io.kappa[v][g], io.phase[v][g], __longlong_as_double((long long)io.cell_mask[v][g]));
  }
  int4 tail;
  tail.x = (int)(unsigned short)bb.x | ((int)bb.y << 16);
  tail.y = (int)(unsigned short)bb.z | ((int)bb.w << 16);
  tail.z = p;
  tail.w = g;
  if (!live) return;
  double4* r = reinterpret_cast<double4*>(rec + i);
  r[0] = r0;
  r[1] = r1;
  reinterpret_cast<int4*>(rec + i)[4] = tail;
}

// depth-segment work items: each tile list is cut into segments of at most
// seg_len Gaussians; items are tile-major, segment-minor.  One block per view.
struct ItemsIO {
  int32_t* range[kMaxBatch];
  int32_t* items[kMaxBatch];
  int32_t* tile_first[kMaxBatch];
  int32_t* n_items[kMaxBatch];
  const int32_t* n_dev[kMaxBatch];
};

__global__ void __launch_bounds__(1024) k_range_init(const __grid_constant__ ItemsIO io, int n_tiles) {
  int32_t* range = io.range[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n_tiles; i += gridDim.x * blockDim.x) range[i] = -1;
}

__global__ void __launch_bounds__(1024) k_make_items(const __grid_constant__ ItemsIO io, int n_tiles, int seg_len,
                                                     int max_items, int64_t n_cap) {
  __shared__ int32_t tmp[32];
  const int v = blockIdx.x;
  int32_t* range = io.range[v];
  int32_t* items = io.items[v];
  int32_t* tile_first = io.tile_first[v];
  // empty tiles (range still -1): [s, s] with s = start of the next non-empty
  // tile, or the pair count -- a suffix min over tiles, chunks last to first
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t after = (int32_t)eff_count(n_cap, io.n_dev[v]);
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
          items[4 * it + 3] = it;   // overwritten below with the processing order
        }
      }
    }
    carry += total;
  }
  // processing order (column 3): segment-major -- every tile's first
  // segment, then every second segment, ... -- so a persistent walk starts
  // the heavy first segments (all rays live) in its first wave and the light
  // deep ones (most rays terminated) fill the tail.  Row c holds the item of
  // the c-th claim; position of (tile t, segment k) = off[k] + #(tiles
  // before t with more than k segments), from per-warp ballot counts.
  // Beyond kOrdSeg segments or kOrdWarps * 32 tiles: identity order.
  {
    constexpr int kOrdSeg = 64, kOrdWarps = 128;
    __shared__ int32_t s_cnt[kOrdSeg][kOrdWarps];
    __shared__ int32_t s_off[kOrdSeg + 1];
    __shared__ int32_t s_max;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += 1024)
      atomicMax(&s_max, (range[2 * t + 1] - range[2 * t] + seg_len - 1) / seg_len);
    __syncthreads();
    const int32_t maxseg = s_max;
    const int n_chunks = (n_tiles + 1023) / 1024;
    if (carry <= max_items && maxseg <= kOrdSeg && n_chunks * 32 <= kOrdWarps) {
      for (int c = 0; c < n_chunks; ++c) {
        const int t = c * 1024 + (int)threadIdx.x;
        const int32_t ns = t < n_tiles ? (range[2 * t + 1] - range[2 * t] + seg_len - 1) / seg_len : 0;
        for (int k = 0; k < maxseg; ++k) {
          const uint32_t b = __ballot_sync(0xffffffffu, ns > k);
          if (lane == 0) s_cnt[k][c * 32 + warp] = __popc(b);
        }
      }
      __syncthreads();
      if (threadIdx.x < 32) {   // off[k] = sum of all tiles' counts of segments < k
        int32_t run = 0;
        for (int k = 0; k < maxseg; ++k) {
          int32_t part = 0;
          for (int w = (int)threadIdx.x; w < n_chunks * 32; w += 32) part += s_cnt[k][w];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
          if (threadIdx.x == 0) s_off[k] = run;
          run += part;
        }
      }
      __syncthreads();
      for (int c = 0; c < n_chunks; ++c) {
        const int t = c * 1024 + (int)threadIdx.x;
        const int32_t ns = t < n_tiles ? (range[2 * t + 1] - range[2 * t] + seg_len - 1) / seg_len : 0;
        const int gw = c * 32 + warp;
        int32_t wmax = ns;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) wmax = max(wmax, __shfl_xor_sync(0xffffffffu, wmax, off));
        for (int k = 0; k < wmax; ++k) {
          const uint32_t b = __ballot_sync(0xffffffffu, ns > k);
          if (ns > k) {
            int32_t before = 0;
            for (int w = 0; w < gw; ++w) before += s_cnt[k][w];
            items[4 * (s_off[k] + before + __popc(b & ((1u << lane) - 1u))) + 3] = tile_first[t] + k;
          }
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    io.n_items[v][0] = carry < max_items ? carry : max_items;
    if (carry > max_items) io.n_items[v][1] = 1;
  }
}

// Workspace of a binning batch (plane lists of nv views, pair capacity cap).
static size_t fused_ws_bytes(int64_t n, int nv) {
  return align_up(sizeof(uint32_t)) + align_up(8 * (size_t)nv * ((n + kEmitTile - 1) / kEmitTile));
}

static size_t bin_ws_bytes(int64_t n, int64_t cap, int nv) {
  return std::max(scan_ws_bytes(n, nv), fused_ws_bytes(n, nv)) + align_up(sizeof(uint32_t) * (size_t)nv * cap) +
         radix_ws_bytes(cap, nv);
}

// Count + emit + tile sort + gather + work items for nv views of one plane.
// offsets[v]: (n+1) caller arrays receiving the per-view pair offsets.
int launch_bin_batch(int nv, const sdgr_projection* projs, const sdgr_view* views, int plane,
                     const int32_t* const* orders, int32_t* const* offsets, sdgr_tiles* tls, bool count,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
  if (nv < 1 || nv > kMaxBatch) return SDGR_ERR_INVALID;
  const int64_t n = projs[0].n, cap = tls[0].n_pairs;
  const sdgr_tiles& t0 = tls[0];
  for (int v = 1; v < nv; ++v)
    if (projs[v].n != n || tls[v].n_pairs != cap || tls[v].n_tiles != t0.n_tiles ||
        tls[v].tiles_x != t0.tiles_x || tls[v].device_count != t0.device_count || tls[v].plane != t0.plane)
      return SDGR_ERR_INVALID;
  if (ws_bytes < bin_ws_bytes(n, std::max<int64_t>(cap, 1), nv)) return SDGR_ERR_CAPACITY;
  char* p = static_cast<char*>(ws);
  void* scan_ws = p; p += std::max(scan_ws_bytes(n, nv), fused_ws_bytes(n, nv));
  uint32_t* keys = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * (size_t)nv * std::max<int64_t>(cap, 1));
  const RadixWs r = radix_layout(p, std::max<int64_t>(cap, 1), nv);

  // fused count + emit when every view has emit rows (multi-view steps)
  bool fused = count;
  for (int v = 0; v < nv; ++v) fused = fused && (plane == 0 ? projs[v].comp.emit : projs[v].img.emit) != nullptr;
  if (count && !fused) {
    ScanIO sio;
    for (int v = 0; v < nv; ++v) {
      const sdgr_plane& pl = plane == 0 ? projs[v].comp : projs[v].img;
      sio.ntiles[v] = pl.n_tiles;
      sio.order[v] = orders ? orders[v] : nullptr;
      sio.out[v] = offsets[v];
    }
    const int rc = scan_counts_batch(sio, nv, n, scan_ws, st);
    if (rc != SDGR_OK) return rc;
  }
  ItemsIO iio;
  for (int v = 0; v < nv; ++v) {
    iio.range[v] = tls[v].tile_range;
    iio.items[v] = tls[v].items;
    iio.tile_first[v] = tls[v].tile_first;
    iio.n_items[v] = tls[v].n_items;
    // device-side pair count = offsets[n] (the scan's total) in capacity mode
    iio.n_dev[v] = tls[v].device_count ? offsets[v] + n : nullptr;
  }
  k_range_init<<<dim3((unsigned)std::min(8, (2 * t0.n_tiles + 1023) / 1024), nv), 1024, 0, st>>>(iio, t0.n_tiles);
  note_launch();
  int bits = 1;
  while ((1 << bits) < t0.n_tiles) ++bits;
  const int npass = (bits + 7) / 8;
  if (npass > kMaxPass) return SDGR_ERR_INVALID;
  if (cap > 0 && cudaMemsetAsync(r.hist, 0, r.zero_bytes, st) != cudaSuccess) return SDGR_ERR_CUDA;
  EmitIO eio;
  for (int v = 0; v < nv; ++v) {
    eio.pl[v] = plane == 0 ? projs[v].comp : projs[v].img;
    eio.order[v] = orders ? orders[v] : nullptr;
    eio.offsets[v] = offsets[v];
    eio.keys[v] = cap > 0 ? keys + (size_t)v * cap : nullptr;
    eio.vals[v] = tls[v].pre_prim;
    eio.pair_start[v] = tls[v].pair_start;
    eio.overflow[v] = tls[v].n_items + 1;  // sticky until the caller clears it
  }
  if (fused) {
    FusedEmitIO fio;
    for (int v = 0; v < nv; ++v) {
      const sdgr_plane& pl = plane == 0 ? projs[v].comp : projs[v].img;
      fio.erow[v] = reinterpret_cast<const ulonglong2*>(pl.emit);
      fio.ntiles[v] = pl.n_tiles;
      fio.uv[v] = pl.uv ? pl.uv : pl.packed;
      fio.uv_stride[v] = pl.uv ? 2 : 8;
      fio.inv_cov[v] = pl.inv_cov;
      fio.order[v] = eio.order[v];
      fio.offsets[v] = offsets[v];
      fio.keys[v] = eio.keys[v];
      fio.vals[v] = eio.vals[v];
      fio.pair_start[v] = eio.pair_start[v];
      fio.overflow[v] = eio.overflow[v];
    }
    const int64_t nblk = (n + kEmitTile - 1) / kEmitTile;
    uint32_t* ticket = static_cast<uint32_t*>(scan_ws);
    unsigned long long* status =
        reinterpret_cast<unsigned long long*>(static_cast<char*>(scan_ws) + align_up(sizeof(uint32_t)));
    if (cudaMemsetAsync(scan_ws, 0, fused_ws_bytes(n, nv), st) != cudaSuccess) return SDGR_ERR_CUDA;
    {
      KernelTimer kt(SDGR_K_EMIT, st);
      k_count_emit<<<(unsigned)(nblk * nv), 256, 0, st>>>(fio, nv, n, nblk, t0.tiles_x, views[0].cutoff, cap,
                                                           cap > 0 ? r.hist : nullptr, npass, status, ticket);
    }
  } else {
    KernelTimer kt(SDGR_K_EMIT, st);
    k_emit_pairs<<<dim3(stride_blocks(n, nv, 8), nv), 256, 0, st>>>(eio, n, t0.tiles_x, views[0].cutoff, cap,
                                                                 cap > 0 ? r.hist : nullptr, npass);
  }
  note_launch();
  if (cap > 0) {
    SortIO sio;
    for (int v = 0; v < nv; ++v) {
      sio.kin[v] = keys + (size_t)v * cap;
      sio.vin[v] = nullptr;
      sio.kout[v] = tls[v].pair_tile;
      sio.vout[v] = reinterpret_cast<uint32_t*>(tls[v].pair_pos);
      sio.n_dev[v] = iio.n_dev[v];
    }
    // stable by tile; values = pre-sort positions (iota)
    int rc = radix_passes(sio, true, nv, cap, npass, r, st);
    if (rc != SDGR_OK) return rc;
    GatherIO gio;
    for (int v = 0; v < nv; ++v) {
      const sdgr_plane& pl = plane == 0 ? projs[v].comp : projs[v].img;
      gio.pos[v] = tls[v].pair_pos;
      gio.pre[v] = tls[v].pre_prim;
      gio.n_dev[v] = iio.n_dev[v];
      gio.prim[v] = tls[v].pair_prim;
      gio.uv[v] = pl.uv;
      gio.inv_cov[v] = pl.inv_cov;
      gio.bbox[v] = pl.bbox;
      gio.cell_mask[v] = pl.cell_mask;
      gio.kappa[v] = projs[v].kappa;
      gio.phase[v] = projs[v].phase;
      gio.packed[v] = plane == 0 ? pl.packed : nullptr;
      gio.erow[v] = reinterpret_cast<const ulonglong2*>(pl.emit);
      gio.rec[v] = plane == 0 ? tls[v].pair_rec : nullptr;
      gio.keys[v] = tls[v].pair_tile;
      gio.range[v] = tls[v].tile_range;
      gio.n_items[v] = tls[v].n_items;
      gio.n_tiles[v] = tls[v].n_tiles;
    }
    {
      KernelTimer kt(SDGR_K_GATHER, st);
      k_gather_prim<<<dim3((unsigned)((cap + 255) / 256), nv), 256, 0, st>>>(gio, cap);
    }
    note_launch();
  }
  k_make_items<<<nv, 1024, 0, st>>>(iio, t0.n_tiles, t0.seg_len, t0.max_items, cap);
  note_launch();
  return check_launch();
}

// Counting alone (sdgr_count_pairs): offsets per view.
int launch_count_batch(int nv, const int32_t* const* ntiles, const int32_t* const* orders, int64_t n,
                       int32_t* const* offsets, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (nv < 1 || nv > kMaxBatch) return SDGR_ERR_INVALID;
  if (ws_bytes < scan_ws_bytes(n, nv)) return SDGR_ERR_CAPACITY;
  ScanIO sio;
  for (int v = 0; v < nv; ++v) {
    sio.ntiles[v] = ntiles[v];
    sio.order[v] = orders ? orders[v] : nullptr;
    sio.out[v] = offsets[v];
  }
  return scan_counts_batch(sio, nv, n, ws, st);
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

struct DepthIO {
  const uint64_t* key[kMaxBatch];
  int32_t* order[kMaxBatch];
};

__device__ __forceinline__ double key_to_depth(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// range[2v] = min visible key, range[2v+1] = ~max visible key (both by
// atomicMin so one 0xff memset initialises them).  Each thread reads
// kKeyIpt keys (pairs of 16-byte loads, block-strided) before reducing.
constexpr int kKeyIpt = 16;

__global__ void __launch_bounds__(256) k_key_range(const __grid_constant__ DepthIO io, int64_t n,
                                                   unsigned long long* range_all) {
  const int v = blockIdx.y;
  const uint64_t* key = io.key[v];
  unsigned long long lo = ~0ull, hi = 0ull;
  const int64_t b0 = (int64_t)blockIdx.x * 256 * kKeyIpt;
  uint64_t k[kKeyIpt];
#pragma unroll
  for (int j = 0; j < kKeyIpt / 2; ++j) {
    const int64_t i = b0 + 2 * (j * 256 + threadIdx.x);
    if (i + 1 < n) {
      const ulonglong2 kk = reinterpret_cast<const ulonglong2*>(key + i)[0];
      k[2 * j] = kk.x; k[2 * j + 1] = kk.y;
    } else {
      k[2 * j] = i < n ? key[i] : ~0ull;
      k[2 * j + 1] = ~0ull;
    }
  }
#pragma unroll
  for (int j = 0; j < kKeyIpt; ++j)
    if (k[j] != ~0ull) {
      lo = k[j] < lo ? k[j] : lo;
      hi = k[j] > hi ? k[j] : hi;
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
    if (lo != ~0ull) atomicMin(range_all + 2 * v, lo);
    if (hi != 0ull) atomicMin(range_all + 2 * v + 1, ~hi);
  }
}

// 24-bit keys + their three digit histograms
__global__ void __launch_bounds__(256) k_key32(const __grid_constant__ DepthIO io, int64_t n, int64_t ks,
                                               const unsigned long long* range_all, uint32_t* k32_all,
                                               uint32_t* hist) {
  __shared__ uint32_t sh[kMaxPass][256];
  BlockHist bh{sh};
  bh.clear();
  const int v = blockIdx.y;
  const uint64_t* key = io.key[v];
  uint32_t* k32 = k32_all + (size_t)v * ks;
  const double dmin = key_to_depth(range_all[2 * v]), dmax = key_to_depth(~range_all[2 * v + 1]);
  const double span = dsub(dmax, dmin);
  const double scale = span > 0.0 ? (double)kKeyMax / span : 0.0;
  const int64_t b0 = (int64_t)blockIdx.x * 256 * kKeyIpt;
  uint64_t k[kKeyIpt];
#pragma unroll
  for (int j = 0; j < kKeyIpt / 2; ++j) {
    const int64_t i = b0 + 2 * (j * 256 + threadIdx.x);
    if (i + 1 < n) {
      const ulonglong2 kk = reinterpret_cast<const ulonglong2*>(key + i)[0];
      k[2 * j] = kk.x; k[2 * j + 1] = kk.y;
    } else {
      k[2 * j] = i < n ? key[i] : ~0ull;
      k[2 * j + 1] = ~0ull;
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kKeyIpt / 2; ++j) {
    const int64_t i = b0 + 2 * (j * 256 + threadIdx.x);
    uint32_t q2[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      uint32_t q32 = kKeyInvisible;
      if (k[2 * j + e] != ~0ull) {
        double q = 0.0;
        if (span > 0.0) q = dmul(dsub(key_to_depth(k[2 * j + e]), dmin), scale);
        q32 = (uint32_t)fmin(fmax(q, 0.0), (double)kKeyMax);
      }
      q2[e] = q32;
    }
    if (i + 1 < n) {
      reinterpret_cast<uint2*>(k32 + i)[0] = make_uint2(q2[0], q2[1]);
      bh.add(q2[0], kMaxPass);
      bh.add(q2[1], kMaxPass);
    } else if (i < n) {
      k32[i] = q2[0];
      bh.add(q2[0], kMaxPass);
    }
  }
  __syncthreads();
  bh.flush(hist + (size_t)v * kHistStride, kMaxPass);
}

// Runs of equal k32 (~10 % of the keys on c4, almost all of length 2-3): the
// last radix pass wrote its order to `tmp`; one thread per position copies it
// to `order`, except that a member of a run of L <= kRunPar entries computes
// its rank under (64-bit key, index) against the L - 1 others (independent,
// L1-resident loads) and lands at run start + rank.  Each thread looks at
// most kRunPar positions either way, so no run costs more than O(L kRunPar).
// Longer runs (many equal depths, or one far outlier squeezing the visible
// depths into few buckets) are listed by their head and sorted by
// k_sort_long_runs.
constexpr int kRunPar = 64;

__global__ void __launch_bounds__(256) k_fix_runs(const uint32_t* k32s_all, const uint32_t* tmp_all, int64_t ks,
                                                  const __grid_constant__ DepthIO io, int64_t n,
                                                  unsigned long long* lr_count, int64_t* lr_start, int64_t lr_cap) {
  const int v = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* k32s = k32s_all + (size_t)v * ks;
  const uint32_t* tmp = tmp_all + (size_t)v * ks;
  int32_t* order = io.order[v];
  const uint32_t k = k32s[i];
  const int32_t g = (int32_t)tmp[i];
  if (k == kKeyInvisible) { order[i] = g; return; }   // invisible tail: order irrelevant
  int64_t s = i, e = i + 1;
  while (s > 0 && i - s < kRunPar && k32s[s - 1] == k) --s;
  while (e < n && e - i <= kRunPar && k32s[e] == k) ++e;
  const bool open_lo = s > 0 && k32s[s - 1] == k, open_hi = e < n && k32s[e] == k;
  if (open_lo || open_hi || e - s > kRunPar) {       // long run: index order now, sorted later
    order[i] = g;
    if (!open_lo && s == i) {
      const unsigned long long j = atomicAdd(lr_count + v, 1ull);
      if ((int64_t)j < lr_cap) lr_start[(int64_t)v * lr_cap + (int64_t)j] = i;
    }
    return;
  }
  if (e - s == 1) { order[i] = g; return; }
  const uint64_t* key = io.key[v];
  const uint64_t kg = key[g];
  int rank = 0;
  for (int64_t j = s; j < e; ++j) {
    const int32_t h = (int32_t)tmp[j];
    const uint64_t kh = key[h];
    rank += (j != i && (kh < kg || (kh == kg && h < g))) ? 1 : 0;
  }
  order[s + rank] = g;
}

// One CTA per long run (grid-stride over the view's list): a block-serial
// stable LSD radix sort of the run's scene indices by the 64-bit depth key,
// one 8-bit pass per key byte that varies within the run (the input is in
// index order, so equal keys keep index order: (depth, index) exactly).
// Ping-pong between order[] and `scratch` (the view's free 24-bit key array).
__global__ void __launch_bounds__(256) k_sort_long_runs(const uint32_t* k32s_all, int64_t ks,
                                                        const __grid_constant__ DepthIO io, int64_t n,
                                                        const unsigned long long* lr_count, const int64_t* lr_start,
                                                        int64_t lr_cap, uint32_t* scratch_all) {
  __shared__ int32_t base[256];
  __shared__ unsigned long long s_or[8], s_and[8];
  const int v = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t* k32s = k32s_all + (size_t)v * ks;
  int32_t* order = io.order[v];
  int32_t* scratch = reinterpret_cast<int32_t*>(scratch_all + (size_t)v * ks);
  const uint64_t* key = io.key[v];
  const int64_t cnt = min((int64_t)lr_count[v], lr_cap);
  for (int64_t r = blockIdx.x; r < cnt; r += gridDim.x) {
    const int64_t s = lr_start[(int64_t)v * lr_cap + r];
    const uint32_t k = k32s[s];
    int64_t e = s;
    while (true) {   // run end: equal keys form a prefix of every 256-wide window
      const int64_t p = e + tid;
      const int same = __syncthreads_count(p < n && k32s[p] == k);
      e += same;
      if (same < 256) break;
    }
    // bits that vary within the run
    unsigned long long o = 0ull, a = ~0ull;
    for (int64_t p = s + tid; p < e; p += 256) {
      const uint64_t kk = key[order[p]];
      o |= kk;
      a &= kk;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      o |= __shfl_xor_sync(0xffffffffu, o, off);
      a &= __shfl_xor_sync(0xffffffffu, a, off);
    }
    if (lane == 0) { s_or[warp] = o; s_and[warp] = a; }
    __syncthreads();
    unsigned long long vary = 0ull;
    for (int w = 0; w < 8; ++w) vary |= s_or[w] ^ s_and[w];
    int32_t* src = order;
    int32_t* dst = scratch;
    for (int b = 0; b < 8; ++b) {
      if (((vary >> (8 * b)) & 255ull) == 0) continue;
      base[tid] = 0;
      __syncthreads();
      for (int64_t p = s + tid; p < e; p += 256) atomicAdd(&base[(key[src[p]] >> (8 * b)) & 255], 1);
      __syncthreads();
      if (tid == 0) {   // exclusive scan of the 256 digit counts (offsets from s)
        int run = 0;
        for (int d = 0; d < 256; ++d) { const int c = base[d]; base[d] = run; run += c; }
      }
      __syncthreads();
      for (int64_t t0 = s; t0 < e; t0 += 256) {
        const int64_t p = t0 + tid;
        const bool ok = p < e;
        const int32_t gi = ok ? src[p] : 0;
        const int d = ok ? (int)((key[gi] >> (8 * b)) & 255) : -1;
        for (int w = 0; w < 8; ++w) {          // warps in order, lanes in order: stable
          if (warp == w) {
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const int before = __popc(peers & ((1u << lane) - 1u));
            const int leader = __ffs(peers) - 1;
            int b0 = 0;
            if (ok && lane == leader) b0 = base[d];
            b0 = __shfl_sync(0xffffffffu, b0, leader);
            if (ok) dst[s + b0 + before] = gi;
            __syncwarp();
            if (ok && lane == leader) base[d] = b0 + __popc(peers);
          }
          __syncthreads();
        }
      }
      int32_t* t = src; src = dst; dst = t;
      __syncthreads();
    }
    if (src != order)
      for (int64_t p = s + tid; p < e; p += 256) order[p] = src[p];
    __syncthreads();
  }
}

// per-view stride of the 24-bit key arrays (keeps uint2 stores aligned)
static int64_t key_stride(int64_t n) { return (n + 63) & ~int64_t(63); }

static int64_t long_run_cap(int64_t n) { return n / (kRunPar + 1) + 1; }

static size_t depth_ws_bytes(int64_t n, int nv) {
  return align_up(16 * (size_t)nv) + 3 * align_up(sizeof(uint32_t) * (size_t)nv * key_stride(n)) +
         align_up(8 * (size_t)nv) + align_up(8 * (size_t)nv * long_run_cap(n)) + radix_ws_bytes(n, nv);
}

int launch_depth_order_batch(int nv, const sdgr_projection* projs, int32_t* const* orders, void* ws,
                             size_t ws_bytes, cudaStream_t st) {
  if (nv < 1 || nv > kMaxBatch) return SDGR_ERR_INVALID;
  const int64_t n = projs[0].n;
  for (int v = 1; v < nv; ++v)
    if (projs[v].n != n) return SDGR_ERR_INVALID;
  if (ws_bytes < depth_ws_bytes(n, nv)) return SDGR_ERR_CAPACITY;
  char* p = static_cast<char*>(ws);
  unsigned long long* range = reinterpret_cast<unsigned long long*>(p); p += align_up(16 * (size_t)nv);
  const int64_t ks = key_stride(n);
  uint32_t* k32 = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * (size_t)nv * ks);
  uint32_t* k32s = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * (size_t)nv * ks);
  uint32_t* tmp = reinterpret_cast<uint32_t*>(p); p += align_up(sizeof(uint32_t) * (size_t)nv * ks);
  unsigned long long* lr_count = reinterpret_cast<unsigned long long*>(p); p += align_up(8 * (size_t)nv);
  const int64_t lr_cap = long_run_cap(n);
  int64_t* lr_start = reinterpret_cast<int64_t*>(p); p += align_up(8 * (size_t)nv * lr_cap);
  const RadixWs r = radix_layout(p, n, nv);
  DepthIO dio;
  for (int v = 0; v < nv; ++v) {
    if (reinterpret_cast<uintptr_t>(projs[v].depth_key) & 15) return SDGR_ERR_INVALID;  // 16-byte loads
    dio.key[v] = projs[v].depth_key;
    dio.order[v] = orders[v];
  }
  if (cudaMemsetAsync(range, 0xff, 16 * (size_t)nv, st) != cudaSuccess ||
      cudaMemsetAsync(lr_count, 0, 8 * (size_t)nv, st) != cudaSuccess ||
      cudaMemsetAsync(r.hist, 0, r.zero_bytes, st) != cudaSuccess)
    return SDGR_ERR_CUDA;
  const unsigned kb = (unsigned)((n + 256 * kKeyIpt - 1) / (256 * kKeyIpt));
  k_key_range<<<dim3(kb, nv), 256, 0, st>>>(dio, n, range);
  k_key32<<<dim3(kb, nv), 256, 0, st>>>(dio, n, ks, range, k32, r.hist);
  note_launch(2);
  SortIO sio;
  for (int v = 0; v < nv; ++v) {
    sio.kin[v] = k32 + (size_t)v * ks;
    sio.vin[v] = nullptr;
    sio.kout[v] = k32s + (size_t)v * ks;
    sio.vout[v] = tmp + (size_t)v * ks;   // k_fix_runs moves it to orders[v]
    sio.n_dev[v] = nullptr;
  }
  const int rc = radix_passes(sio, true, nv, n, kMaxPass, r, st);
  if (rc != SDGR_OK) return rc;
  k_fix_runs<<<dim3((unsigned)((n + 255) / 256), nv), 256, 0, st>>>(k32s, tmp, ks, dio, n, lr_count, lr_start,
                                                                      lr_cap);
  // (normally no long runs: the CTAs read a zero count and exit)
  k_sort_long_runs<<<dim3(8, nv), 256, 0, st>>>(k32s, ks, dio, n, lr_count, lr_start, lr_cap, k32);
  note_launch(2);
  return check_launch();
}

// ------------------------------------------------- generic key sort --------
// Stable sort of n 32-bit keys (bits [0, bits)) with their input positions:
// keys_out ascending, perm_out[i] = input index.  Used by the evaluation grid
// (eval.cu).
__global__ void __launch_bounds__(256) k_key_hist(const uint32_t* keys, int64_t n, int npass, uint32_t* hist) {
  __shared__ uint32_t sh[kMaxPass][256];
  BlockHist bh{sh};
  bh.clear();
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bh.add(keys[i], npass);
  __syncthreads();
  bh.flush(hist, npass);
}

size_t sort_u32_ws_bytes(int64_t n) { return radix_ws_bytes(n < 1 ? 1 : n, 1) + 4096; }

int sort_u32(const uint32_t* keys, int64_t n, int bits, uint32_t* keys_out, uint32_t* perm_out, void* ws,
             size_t ws_bytes, cudaStream_t st) {
  if (n <= 0) return SDGR_OK;
  const int npass = (bits + 7) / 8;
  if (npass < 1 || npass > kMaxPass) return SDGR_ERR_INVALID;
  if (ws_bytes < sort_u32_ws_bytes(n)) return SDGR_ERR_CAPACITY;
  char* p = static_cast<char*>(ws);
  const RadixWs r = radix_layout(p, n, 1);
  if (cudaMemsetAsync(r.hist, 0, r.zero_bytes, st) != cudaSuccess) return SDGR_ERR_CUDA;
  k_key_hist<<<stride_blocks(n, 1, 2), 256, 0, st>>>(keys, n, npass, r.hist);
  note_launch();
  SortIO io;
  io.kin[0] = keys;
  io.vin[0] = nullptr;
  io.kout[0] = keys_out;
  io.vout[0] = perm_out;
  io.n_dev[0] = nullptr;
  return radix_passes(io, true, 1, n, npass, r, st);
}

size_t batch_ws_bytes(int64_t n, int64_t max_pairs, int nv) {
  return std::max(depth_ws_bytes(n, nv), bin_ws_bytes(n, max_pairs, nv)) + 4096;
}

}  // namespace sdgr
