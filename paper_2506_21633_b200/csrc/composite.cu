// composite.cu — K6/K7/K9: compositing on the computation plane and the
// imaging-plane splat.
//
// Order-INdependent sums run as streaming kernels with deterministic
// fixed-point accumulation (integer adds are associative, so the result does
// not depend on thread timing):
//   k_segsum   per depth segment of a tile, the optical depth each ray
//              accumulates (sum of tau), global u64 fixed-point REDs;
//   k_splat    image[p] = sum_g w I_g, Gaussian-parallel, global u64 REDs.
// Order-DEpendent passes are tile walks.  A work item is one depth segment
// (<= seg_len Gaussians) of one 16x16 tile list; a persistent CTA of 256
// threads pulls items from an atomic counter.  Thread r owns ray r of the tile
// for the order-dependent steps; thread j owns Gaussian j of the chunk:
//   P0  thread j loads the packed record of pair j (coalesced) and derives its
//       256-bit in-tile member mask from the 8x8 cell window K1 stored (the
//       exact FP64 membership is reused); bits go into a cell-major bitmap.
//   P1  thread r counts its ray's live members; a block scan lays every live
//       (ray, member) pair out in a flat shared array in ray-major,
//       depth-minor order -- exactly the reference's per-ray walk order.
//   P2  thread j places its own live member pairs (slot, Gaussian, ray) in
//       the flat array; then w = exp(-q) and tau = kappa w are evaluated
//       pair-parallel over the slots (<= capacity / 256 per thread, balanced
//       whatever the per-Gaussian member counts).
//   P3  log-transmittance prefix and early termination: a block segmented
//       scan over the ray runs (S at a pair = the ray's S at the sub-chunk
//       start + the run's exclusive sum; SDGR_WALK_P3_SCAN=0: thread r walks
//       its run).
//   P4  flat pair-parallel pass: T = e^-S, 1 - e^-tau, contributions.
//   P5  thread r: downstream suffix sums (backward only; adds only).
//   P7  thread j reduces its own pairs in cell order into ONE partial record
//       per (tile, Gaussian) pair, indexed by the pair's pre-sort position:
//       no atomics, fixed order => deterministic.
// A chunk whose live pairs exceed the flat array is processed in sub-chunks
// of consecutive Gaussians (ray state carries over).
//
// Modes (reference stage they replace):
//   k_segsum  segment optical-depth sums        (forward.py:182-187, cumsum)
//   kContrib  per-pair contributions -> I_g      (forward.py:188-192)
//   k_splat   image = sum_g w I_g                (forward.py:227-240)
//   kGSum     segment sums of g*contrib          (backward.py:129-139)
//   kGrad     reverse-recurrence gradients       (backward.py:122-148)
// Depth segments are stitched with per-ray exclusive prefix (forward) /
// suffix (backward) scans over a tile's items, in FP64.
//
// Early ray termination: a ray stops once its log-transmittance S exceeds
// s_stop (contributions < e^-s_stop * P).  s_stop = +inf reproduces the
// reference's exhaustive walk.
#include <numeric>

#include "common.cuh"

namespace sdgr {

enum WalkMode { kContrib = 1, kGSum = 3, kGrad = 4 };
// Persistent walk grids: SDGR_WALK_GRID_DIV = 1 fills every SM's resident
// CTA slots with one view's walk; > 1 leaves room for the walks of views on
// other streams to run alongside (A/B knob for the multi-view step).
// Flat live-pair capacity of a walk sub-chunk (and the replay's descriptor
// buffer), chosen per binning from the pair capacity (big_walk below):
//   small config: 1024 entries, walk / kGrad at 4 CTAs/SM, kGSum at 6 --
//     best for large views in the concurrent 8-lane step (c4 1365 -> 1416
//     views/s): the smaller footprints let more CTAs of the co-running lanes
//     stay resident, although a lone walk launch gets slower (more
//     sub-chunks);
//   big config: 2048 entries, walk / kGrad at 3 CTAs/SM, kGSum at 4 -- small
//     views (c2, the 10k-100k points of the c5 sweep), whose walks are short
//     enough that the extra sub-chunks dominate (profiles/ROUND2.md).
#ifndef SDGR_WALK_CAP
#define SDGR_WALK_CAP 1024
#endif
#ifndef SDGR_WALK_CAP_BIG
#define SDGR_WALK_CAP_BIG 2048
#endif
// views whose pair capacity is at most this use the big config
#ifndef SDGR_BIG_WALK_PAIRS
#define SDGR_BIG_WALK_PAIRS 400000
#endif
static bool big_walk(const sdgr_tiles& t) { return t.n_pairs <= (int64_t)SDGR_BIG_WALK_PAIRS; }
// 1: walk P0 reads the chunk's 80-byte pair records from shared memory,
// where a cp.async.bulk (TMA engine, mbarrier completion) issued during the
// previous chunk put them.  Measured slower and off by default (c4, 1367
// views/s without; with it 1318 at 2 CTAs/SM, 1344 with the flat capacity
// cut to 1408 to keep 3 CTAs/SM, vs 1360 for that capacity without: the
// record loads are not P0's cost; profiles/ROUND2.md).  The full GPU test
// suite passes with it on.
#ifndef SDGR_WALK_BULK
#define SDGR_WALK_BULK 0
#endif
#ifndef SDGR_DESC_CACHE
#define SDGR_DESC_CACHE 256
#endif
constexpr int kDescCache = SDGR_DESC_CACHE;
// Item claim order of the persistent kernels: 1 = the segment-major order
// k_make_items writes (heavy first segments first), 0 = tile-major item
// order.  c4 (profiles/ROUND2.md): segment-major cuts the lone walk launch
// 9.0 -> 7.75 ms/step (its tail) at -0.3 % views/s in the concurrent step;
// for pass A and the replays it costs 0.5-1 % views/s and is off.
#ifndef SDGR_ORDER_WALK
#define SDGR_ORDER_WALK 1
#endif
#ifndef SDGR_ORDER_SEGSUM
#define SDGR_ORDER_SEGSUM 0
#endif
#ifndef SDGR_ORDER_REPLAY
#define SDGR_ORDER_REPLAY 0
#endif
#ifndef SDGR_WALK_GRID_DIV
#define SDGR_WALK_GRID_DIV 1
#endif
static int persistent_grid(int per_sm) {
  return std::max(1, sm_count() * std::max(per_sm, 1) / SDGR_WALK_GRID_DIV);
}


// fixed point: value * 2^32 in a u64 (values are >= 0)
constexpr double kFix = 4294967296.0;
constexpr double kFixInv = 1.0 / 4294967296.0;
constexpr double kFixMax = 1.0e5;  // per-term clamp: keeps 8192-term sums far from 2^32

template <int MODE, bool kBig>
struct WalkCfg {
  static constexpr int kCap = MODE == kGSum ? 4096 : (kBig ? SDGR_WALK_CAP_BIG : SDGR_WALK_CAP);  // flat pair slots
  static constexpr bool kXY = MODE == kGrad;
  // + the chunk's records, staged by a bulk copy (TMA engine) one chunk ahead
  static constexpr size_t kStage = SDGR_WALK_BULK ? (size_t)kChunk * sizeof(sdgr_pair_rec) : 0;
  static constexpr size_t kSmem = kStage + kCap * (8 + 8 + (kXY ? 16 : 0) + 2);
};
// replay buffer = the walk's flat capacity: one descriptor fits (a 2048
// replay with the 1024 walk: 1416 -> 1383 views/s)
template <bool kBig>
constexpr int replay_cap() { return kBig ? SDGR_WALK_CAP_BIG : SDGR_WALK_CAP; }

struct WalkArgs {
  int n_cols, n_rows, tiles_x;
  double cutoff;
  const sdgr_pair_rec* rec;
  const int32_t* items;
  const int32_t* n_items;
  uint32_t* counter;
  const double* gvec;      // kGSum/kGrad: dL/dI
  double s_stop;
  const double* seg_base;  // exclusive prefix of optical depth per (item, ray)
  const double* seg_g;     // kGrad: this segment's sum of g*contrib
  const double* seg_d;     // kGrad: downstream (later segments) sum of g*contrib
  double* seg_out;         // kGSum: seg_g
  double* partial;         // kContrib: (n_pairs); kGrad: (n_pairs, 8)
  int32_t* status;
  sdgr_replay rp;          // kContrib: live-pair log to write (rp.y1 == nullptr: none)
};

// ---- bulk copy global -> shared with mbarrier completion (one thread issues)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(mbar)) : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  // earlier generic-proxy reads of dst are ordered before the async write
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(mbar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(mbar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(mbar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ sdgr_pair_rec load_rec_smem(const sdgr_pair_rec* p) {
  sdgr_pair_rec r;
  const double2* s = reinterpret_cast<const double2*>(p);
  const double2 a0 = s[0], a1 = s[1], b0 = s[2], b1 = s[3];
  const int4 t = reinterpret_cast<const int4*>(p)[4];
  r.u = a0.x; r.v = a0.y; r.a00 = a1.x; r.a01 = a1.y;
  r.a11 = b0.x; r.kappa = b0.y; r.phase = b1.x; r.cell_mask = (uint64_t)__double_as_longlong(b1.y);
  r.x0 = (int16_t)(t.x & 0xffff); r.x1 = (int16_t)(t.x >> 16);
  r.y0 = (int16_t)(t.y & 0xffff); r.y1 = (int16_t)(t.y >> 16);
  r.pos = t.z; r.prim = t.w;
  return r;
}

// The bits of an 8x8 cell window at (cx0, cy0) (relative to a 16x16 tile)
// that fall inside the tile.
__device__ __forceinline__ uint64_t window_clip(int cx0, int cy0) {
  const int clo = max(0, -cx0), chi = min(7, kTile - 1 - cx0);
  const int rlo = max(0, -cy0), rhi = min(7, kTile - 1 - cy0);
  if (clo > chi || rlo > rhi) return 0ull;
  const uint64_t col8 = ((2ull << chi) - 1ull) & ~((1ull << clo) - 1ull);
  const uint64_t rows = (rhi >= 7 ? ~0ull : ((1ull << (8 * (rhi + 1))) - 1ull)) & ~((1ull << (8 * rlo)) - 1ull);
  return (col8 * 0x0101010101010101ull) & rows;
}

__device__ __forceinline__ sdgr_pair_rec load_rec(const sdgr_pair_rec* p) {
  sdgr_pair_rec r;
  const double2* s = reinterpret_cast<const double2*>(p);
  const double2 a0 = __ldg(s), a1 = __ldg(s + 1), b0 = __ldg(s + 2), b1 = __ldg(s + 3);
  const int4 t = __ldg(reinterpret_cast<const int4*>(p) + 4);
  r.u = a0.x; r.v = a0.y; r.a00 = a1.x; r.a01 = a1.y;
  r.a11 = b0.x; r.kappa = b0.y; r.phase = b1.x; r.cell_mask = (uint64_t)__double_as_longlong(b1.y);
  r.x0 = (int16_t)(t.x & 0xffff); r.x1 = (int16_t)(t.x >> 16);
  r.y0 = (int16_t)(t.y & 0xffff); r.y1 = (int16_t)(t.y >> 16);
  r.pos = t.z; r.prim = t.w;
  return r;
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

// ============================================================ pass A ==========
// Per (segment, ray) fixed-point sums of tau, accumulated with fire-and-forget
// global RED.ADD.U64 (native; integer adds commute, so the sums are exact and
// deterministic); the segment scan converts them back to FP64.
//
// Work is flattened per warp: the 32 lanes' member masks are laid end to end
// (warp scan of their popcounts) and each round of the loop hands one member
// (Gaussian, cell) to every lane, so the exp/RED work runs at full SIMT width
// whatever the per-Gaussian member counts are.

// Member lists: each lane appends its (lane, cell) entries at its exclusive
// offset into a per-warp window of kList slots; windows repeat until the
// warp's total is covered (a lane keeps its not-yet-written bits).
#ifndef SDGR_MEMBER_LIST
#define SDGR_MEMBER_LIST 512
#endif
constexpr int kList = SDGR_MEMBER_LIST;

__device__ __forceinline__ void fill_window(uint64_t mr[4], int& nx, int lim, int lane, uint16_t* list, int B) {
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    uint64_t x = mr[w];
    while (x && nx < lim) {
      const int b = __ffsll((long long)x) - 1;
      x &= x - 1;
      list[nx - B] = (uint16_t)((lane << 8) | (w * 64 + b));
      ++nx;
    }
    mr[w] = x;
  }
}

#ifndef SDGR_MINB_SEGSUM
#define SDGR_MINB_SEGSUM 1
#endif
#ifndef SDGR_MINB_SPLAT
#define SDGR_MINB_SPLAT 1
#endif
__global__ void __launch_bounds__(256, SDGR_MINB_SEGSUM) k_segsum(const sdgr_pair_rec* rec, const int32_t* items,
                                                const int32_t* n_items_p, uint32_t* counter, int tiles_x,
                                                double cutoff, unsigned long long* seg_fx) {
  __shared__ int item_s;
  __shared__ double s_u[kRays], s_v[kRays], s_a0[kRays], s_a1[kRays], s_a2[kRays], s_k[kRays];
  __shared__ uint16_t s_list[8 * kList];
  const int tid = threadIdx.x, lane = tid & 31, wbase = tid & ~31;
  uint16_t* list = s_list + (tid >> 5) * kList;
  const int n_items = *n_items_p;
  while (true) {
    __syncthreads();
    if (tid == 0) item_s = (int)atomicAdd(counter, 1u);
    __syncthreads();
    if (item_s >= n_items) return;
    const int item = SDGR_ORDER_SEGSUM ? items[4 * item_s + 3] : item_s;   // processing order (k_make_items)
    const int4 it = reinterpret_cast<const int4*>(items)[item];
    // a tile's last segment: its optical depth is no later segment's prefix
    // (the scan is exclusive), so pass A skips it -- for a single-segment
    // tile, the whole tile
    if (item + 1 >= n_items || items[4 * (item + 1)] != it.x) continue;
    const int tx = it.x % tiles_x, ty = it.x / tiles_x;
    unsigned long long* acc = seg_fx + (int64_t)item * kRays;
    for (int i0 = it.y; i0 < it.z; i0 += kRays) {
      // small footprints (the common case): the 8x8 window mask K1 stored,
      // clipped to this tile, and the window origin relative to the tile --
      // list entries are made from its bits directly; larger footprints:
      // the 256-bit in-tile mask of the exact per-cell test
      uint64_t m[4] = {0, 0, 0, 0};
      uint64_t wm = 0;
      int cx0 = 0, cy0 = 0;
      if (i0 + tid < it.z) {
        const sdgr_pair_rec r = load_rec(rec + i0 + tid);
        if (r.x0 <= r.x1 && r.y0 <= r.y1 && (r.x1 - r.x0) < 8 && (r.y1 - r.y0) < 8) {
          cx0 = r.x0 - tx * kTile;
          cy0 = r.y0 - ty * kTile;
          wm = r.cell_mask & window_clip(cx0, cy0);
        } else {
          member_mask(r, tx, ty, cutoff, m);
        }
        s_u[tid] = r.u; s_v[tid] = r.v;
        s_a0[tid] = r.a00; s_a1[tid] = r.a01; s_a2[tid] = r.a11; s_k[tid] = r.kappa;
      }
      const int cnt = __popcll(wm) + __popcll(m[0]) + __popcll(m[1]) + __popcll(m[2]) + __popcll(m[3]);
      int incl = cnt;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      int nx = incl - cnt;
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      for (int B = 0; B < tot; B += kList) {
        const int lim = min(tot, B + kList);
        while (wm && nx < lim) {   // window bits -> tile-local cells, in the 256-bit order
          const int b = __ffsll((long long)wm) - 1;
          wm &= wm - 1;
          list[nx - B] = (uint16_t)((lane << 8) | (((cy0 + (b >> 3)) << 4) | (cx0 + (b & 7))));
          ++nx;
        }
        fill_window(m, nx, lim, lane, list, B);
        __syncwarp();
        for (int k = B + lane; k < lim; k += 32) {
          const int e = list[k - B];
          const int j = wbase + (e >> 8), c = e & 255;
          const double dx = dsub((double)(tx * kTile + (c & 15)), s_u[j]);
          const double dy = dsub((double)(ty * kTile + (c >> 4)), s_v[j]);
          const double tau = s_k[j] * exp(-quadform(s_a0[j], s_a1[j], s_a2[j], dx, dy));
          atomicAdd(acc + c, (unsigned long long)__double2ull_rn(fmin(tau, kFixMax) * kFix));
        }
        __syncwarp();
      }
    }
  }
}

// ============================================================ splat ===========
// One thread per Gaussian; its member pixels (imaging-plane cell window K1
// stored) receive w * I_g through global u64 fixed-point REDs.  Small
// footprints (<= 8x8 window) are flattened per warp through a member list
// (as in pass A) so the exp/RED work runs at full SIMT width; larger
// footprints are walked by their own thread.
// Splat fixed point: per view, value * 2^(47 - e) with 2^e > max_g I_g, so
// every term w I <= I_max maps below 2^47 and a pixel can take 2^16 terms at
// the maximum before the u64 sum could wrap; the absolute precision is
// 2^-47 I_max (~7e-15 relative to the brightest Gaussian), whatever the
// scene's brightness.  Integer adds are associative: the image is bitwise
// deterministic.  Non-finite terms saturate at 2^47 (the forward's status
// word has already flagged them).
constexpr double kSplatTop = 140737488355328.0;   // 2^47

__device__ __forceinline__ double splat_scale(const unsigned long long* max_bits) {
  const double M = __longlong_as_double((long long)*max_bits);
  if (!(M > 0.0) || !isfinite(M)) return 1.0;
  int e;
  frexp(M, &e);                 // M < 2^e
  return ldexp(1.0, 47 - e);
}

__device__ __forceinline__ unsigned long long splat_fix(double v, double scale) {
  return (unsigned long long)__double2ull_rn(fmin(v * scale, kSplatTop));
}

__device__ __forceinline__ void splat_add(unsigned long long* acc, int n_az, int iu, int iv, double q, double I,
                                          double scale) {
  atomicAdd(acc + (int64_t)iv * n_az + iu, splat_fix(nexp(-q) * I, scale));
}

// max_g I_g over visible Gaussians as u64 bits (I >= 0: the bit order is the
// value order); grid-stride, one atomic per block
__global__ void __launch_bounds__(256) k_max_intensity(const uint8_t* flags, const double* intensity, int64_t n,
                                                       unsigned long long* max_bits) {
  __shared__ unsigned long long s_max[8];
  unsigned long long b = 0ull;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    const double I = intensity[g];
    if ((flags[g] & SDGR_FLAG_VISIBLE) && I > 0.0 && isfinite(I)) b = max(b, (unsigned long long)__double_as_longlong(I));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) b = max(b, __shfl_down_sync(0xffffffffu, b, off));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) b = max(b, s_max[w]);
    if (b) atomicMax(max_bits, b);
  }
}

// Warps take 32-Gaussian groups in a scattered order: warp w of the grid
// splats group (w * wperm) mod n_groups (wperm coprime to n_groups, ~0.618
// n_groups).  Neighbouring Gaussians of a spatially ordered scene hit the
// same pixels; with consecutive warps on consecutive groups their REDs
// queue on the same L2 addresses (c4: k_splat 4.0 ms/step in the scene's
// own order, 2.6 in a random order).  Loads stay coalesced within a warp.
__global__ void __launch_bounds__(256, SDGR_MINB_SPLAT) k_splat(sdgr_view view, sdgr_plane pl, const uint8_t* flags,
                                               const double* intensity, int64_t n, int64_t wperm,
                                               unsigned long long* acc, const unsigned long long* max_bits) {
  const double scale = splat_scale(max_bits);
  __shared__ double s_u[256], s_v[256], s_a0[256], s_a1[256], s_a2[256], s_I[256];
  __shared__ int32_t s_x[256], s_y[256];
  __shared__ uint16_t s_list[8 * kList];
  const int tid = threadIdx.x, lane = tid & 31, wbase = tid & ~31;
  uint16_t* list = s_list + (tid >> 5) * kList;
  const int64_t n_groups = (n + 31) / 32, wg = (int64_t)blockIdx.x * 8 + (tid >> 5);
  const int64_t g = wg < n_groups ? (wg * wperm) % n_groups * 32 + lane : n;
  uint64_t m[4] = {0, 0, 0, 0};
  bool large = false;
  double2 uv = make_double2(0, 0);
  double4 A = make_double4(0, 0, 0, 0);
  short4 bb = make_short4(0, -1, 0, -1);
  double I = 0.0;
  if (g < n) {   // all rows loaded at once (one round trip), then tested
    const uint8_t fl = flags[g];
    const double Ig = intensity[g];
    const double2 uvg = reinterpret_cast<const double2*>(pl.uv)[g];
    const double4 Ag = reinterpret_cast<const double4*>(pl.inv_cov)[g];
    const short4 bbg = reinterpret_cast<const short4*>(pl.bbox)[g];
    const uint64_t cmg = pl.cell_mask[g];
    if ((fl & SDGR_FLAG_VISIBLE) && Ig != 0.0) {
      I = Ig; uv = uvg; A = Ag; bb = bbg;
      if (bb.x <= bb.y && bb.z <= bb.w) {
        if ((bb.y - bb.x) < 8 && (bb.w - bb.z) < 8) m[0] = cmg;
        else large = true;
      }
    }
  }
  s_u[tid] = uv.x; s_v[tid] = uv.y; s_a0[tid] = A.x; s_a1[tid] = A.y; s_a2[tid] = A.z; s_I[tid] = I;
  s_x[tid] = bb.x; s_y[tid] = bb.z;
  const int cnt = __popcll(m[0]);
  int incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  int nx = incl - cnt;
  const int tot = __shfl_sync(0xffffffffu, incl, 31);
  for (int B = 0; B < tot; B += kList) {
    const int lim = min(tot, B + kList);
    fill_window(m, nx, lim, lane, list, B);
    __syncwarp();
    for (int k0 = B; k0 < lim; k0 += 32) {
      const int k = k0 + lane;
      const bool on = k < lim;
      int64_t pix = 0;
      unsigned long long val = 0ull;
      if (on) {
        const int e = list[k - B];
        const int j = wbase + (e >> 8), b = e & 63;
        const int iu = s_x[j] + (b & 7), iv = s_y[j] + (b >> 3);
        const double q = quadform(s_a0[j], s_a1[j], s_a2[j], dsub((double)iu, s_u[j]), dsub((double)iv, s_v[j]));
        pix = (int64_t)iv * view.n_az + iu;
        val = splat_fix(nexp(-q) * s_I[j], scale);
      }
      // (combining a round's same-pixel terms with MATCH.ANY before the RED
      // was measured slower: 4.0 -> 6.5 ms/step, only ~17 % of the REDs merge)
      if (on) atomicAdd(acc + pix, val);
    }
    __syncwarp();
  }
  if (large) {
    const bool dense = !isfinite(view.cutoff);
    const double cut2 = dmul(view.cutoff, view.cutoff);
    for (int iv = bb.z; iv <= bb.w; ++iv)
      for (int iu = bb.x; iu <= bb.y; ++iu) {
        const double q = quadform(A.x, A.y, A.z, dsub((double)iu, uv.x), dsub((double)iv, uv.y));
        if (dense || q <= cut2) splat_add(acc, view.n_az, iu, iv, q, I, scale);
      }
  }
}

__global__ void __launch_bounds__(256) k_splat_finish(const unsigned long long* acc, int64_t n, double* image) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const double inv = 1.0 / splat_scale(acc + n);
  if (i < n) image[i] = (double)acc[i] * inv;
}

// Segmented inclusive scan across the block: thread t holds cnt <= 8
// consecutive log entries (thread t's before thread t+1's), hd[e] marks the first entry of a run.  On return v[e]
// is the sum of its run up to and including e.  Fixed association order
// (thread-serial, then warp shuffles, then warps in order): deterministic.
// One __syncthreads inside; consecutive calls need a barrier between them.
template <int kE>
__device__ __forceinline__ void block_seg_scan8(double (&v)[kE], const bool (&hd)[kE], int cnt, double* s_agg,
                                                int* s_flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double run = 0.0;
  int any = 0;
#pragma unroll
  for (int e = 0; e < kE; ++e) {
    if (e < cnt) {
      if (hd[e]) { run = v[e]; any = 1; } else { run += v[e]; }
      v[e] = run;
    }
  }
  double a = run;
  int f = any;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double ao = __shfl_up_sync(0xffffffffu, a, off);
    const int fo = __shfl_up_sync(0xffffffffu, f, off);
    if (lane >= off) {
      if (!f) a = ao + a;
      f |= fo;
    }
  }
  double ex = __shfl_up_sync(0xffffffffu, a, 1);
  int exf = __shfl_up_sync(0xffffffffu, f, 1);
  if (lane == 0) { ex = 0.0; exf = 0; }
  if (lane == 31) { s_agg[warp] = a; s_flag[warp] = f; }
  __syncthreads();
  double wc = 0.0;
  for (int w = 0; w < warp; ++w) wc = s_flag[w] ? s_agg[w] : wc + s_agg[w];
  const double carry = exf ? ex : wc + ex;
  bool open = true;
#pragma unroll
  for (int e = 0; e < kE; ++e) {
    if (e < cnt && open) {
      if (hd[e]) open = false;
      else v[e] += carry;
    }
  }
}

// ============================================================ tile walks ======
#ifdef SDGR_WALK_PROFILE
// phase profile of the walks (profiling builds only, profiles/walk_phases.py):
// cycles between the barriers that close each phase, by thread 0 of each CTA
__device__ unsigned long long g_walk_prof[16];
#define WPROF(k)                                                                    \
  do {                                                                              \
    if (threadIdx.x == 0) {                                                         \
      const long long t_ = clock64();                                               \
      atomicAdd(&g_walk_prof[k], (unsigned long long)(t_ - t_prev));                \
      t_prev = t_;                                                                  \
    }                                                                               \
  } while (0)
#else
#define WPROF(k) \
  do {           \
  } while (0)
#endif

#ifndef SDGR_MINB_REPLAY_GSUM_BIG
#define SDGR_MINB_REPLAY_GSUM_BIG 4   // the big-buffer kGSum replay (6: -0.6 %, 8: -5 % on c2)
#endif
#ifndef SDGR_WALK_MINB_BIG
#define SDGR_WALK_MINB_BIG 2   // the big-buffer walk (views up to SDGR_BIG_WALK_PAIRS pairs): no spills (c2 +2 % over 3)
#endif
#ifndef SDGR_WALK_MINB
#define SDGR_WALK_MINB 4
#endif
#ifndef SDGR_WALK_P3_SCAN
#define SDGR_WALK_P3_SCAN 1
#endif
#ifndef SDGR_WALK_P2_FLAT
#define SDGR_WALK_P2_FLAT 1
#endif
template <int MODE, bool kBig>
__global__ void __launch_bounds__(256, kBig ? SDGR_WALK_MINB_BIG : SDGR_WALK_MINB) k_walk(WalkArgs a) {
#ifdef SDGR_WALK_PROFILE
  long long t_prev = clock64();
#endif
  using Cfg = WalkCfg<MODE, kBig>;
  constexpr int kCap = Cfg::kCap;
  __shared__ uint32_t rows[8 * kRays];   // rows[w*256 + r]: bit (j&31) of word w = Gaussian j covers ray r
  __shared__ uint32_t wpre[2 * kRays];   // per ray: byte prefix counts of the masked words
  __shared__ int32_t ray_off[kRays];
  __shared__ uint32_t alive_bits[8];
  __shared__ double su[kChunk], sv[kChunk], sa0[kChunk], sa1[kChunk], sa2[kChunk];
  __shared__ double sk[kChunk], sp[kChunk], sg[MODE == kContrib ? 1 : kChunk];
  __shared__ int32_t scan_tmp[8];
  __shared__ int32_t base_s;
  __shared__ int item_s;
#if SDGR_WALK_P3_SCAN
  __shared__ double s_agg8[8];
  __shared__ int s_flag8[8];
  __shared__ double s_S0[kRays], s_S1[kRays];   // per ray: S at the sub-chunk's start / end
#endif
  extern __shared__ __align__(128) double dyn[];
  sdgr_pair_rec* stage = reinterpret_cast<sdgr_pair_rec*>(dyn);   // the chunk's records (bulk copy)
  double* fw = dyn + Cfg::kStage / 8;                        // w
  double* fs = fw + kCap;                                   // S / contrib / g*contrib / D
  double* fx = fs + kCap;                                   // kGrad: g*T*a*P
  double* fy = fx + (Cfg::kXY ? kCap : 0);                  // kGrad: T*(1-a)
  uint8_t* fj = reinterpret_cast<uint8_t*>(fy + (Cfg::kXY ? kCap : 0));
  uint8_t* fr = fj + kCap;                                  // ray of each slot (replay log)
  __shared__ long long rp_off;
  const bool record = MODE == kContrib && a.rp.y1 != nullptr;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_items = *a.n_items;
  __shared__ __align__(8) uint64_t s_mbar;
  uint32_t parity = 0;
  if (SDGR_WALK_BULK && tid == 0) mbar_init(&s_mbar);
  while (true) {
    __syncthreads();
    if (tid == 0) item_s = (int)atomicAdd(a.counter, 1u);
    __syncthreads();
    WPROF(0);
    if (item_s >= n_items) return;
    const int item = SDGR_ORDER_WALK ? a.items[4 * item_s + 3] : item_s;   // processing order (k_make_items)
    const int4 it = reinterpret_cast<const int4*>(a.items)[item];
    const int tile = it.x, start = it.y, end = it.z;
    const int tx = tile % a.tiles_x, ty = tile / a.tiles_x;
    const int iu = tx * kTile + (tid & 15), iv = ty * kTile + (tid >> 4);
    const bool valid = iu < a.n_cols && iv < a.n_rows;
    const int64_t slot_ray = (int64_t)item * kRays + tid;
    double S = a.seg_base ? a.seg_base[slot_ray] : 0.0, accd = 0.0, rem = 0.0;
    if (MODE == kGrad) rem = a.seg_d[slot_ray] + a.seg_g[slot_ray];
    bool alive = valid && S < a.s_stop;
    bool bad = false;
    int n_desc = 0;

    bool pending = false;   // block-uniform: a bulk copy of chunk `cs` into `stage` is in flight
    int cs = start;
    for (; cs < end; cs += kChunk) {
      if (!__syncthreads_or(alive)) break;
      if (SDGR_WALK_BULK && !pending) {   // an item's first chunk (later ones were prefetched)
        if (tid == 0)
          bulk_load(stage, a.rec + cs, (uint32_t)(min(kChunk, end - cs) * sizeof(sdgr_pair_rec)), &s_mbar);
        pending = true;
      }
      // ---- P0: stage pair j = tid, member mask restricted to live rays,
      //      skip the chunk outright when no Gaussian touches a live ray
#pragma unroll
      for (int w = 0; w < 8; ++w) rows[w * kRays + tid] = 0u;
      {
        const uint32_t ab0 = __ballot_sync(0xffffffffu, alive);
        if (lane == 0) alive_bits[warp] = ab0;
      }
      const int nG = min(kChunk, end - cs);
      const bool have = tid < nG;
      uint64_t gm[4] = {0, 0, 0, 0};
      int pos = 0;
      if (SDGR_WALK_BULK) {
        mbar_wait(&s_mbar, parity);
        parity ^= 1u;
        pending = false;
      }
      if (have) {
        const sdgr_pair_rec r = SDGR_WALK_BULK ? load_rec_smem(stage + tid) : load_rec(a.rec + cs + tid);
        member_mask(r, tx, ty, a.cutoff, gm);
        su[tid] = r.u; sv[tid] = r.v;
        sa0[tid] = r.a00; sa1[tid] = r.a01; sa2[tid] = r.a11;
        sk[tid] = r.kappa; sp[tid] = r.phase;
        if (MODE != kContrib) sg[tid] = a.gvec[r.prim];
        pos = r.pos;
      }
      __syncthreads();
      WPROF(1);
      if (SDGR_WALK_BULK && cs + kChunk < end) {   // the next chunk's records, overlapping this chunk
        if (tid == 0)
          bulk_load(stage, a.rec + cs + kChunk,
                    (uint32_t)(min(kChunk, end - cs - kChunk) * sizeof(sdgr_pair_rec)), &s_mbar);
        pending = true;
      }
#pragma unroll
      for (int w = 0; w < 4; ++w)
        gm[w] &= ((uint64_t)alive_bits[2 * w] | ((uint64_t)alive_bits[2 * w + 1] << 32));
      if (!__syncthreads_or(have && (gm[0] | gm[1] | gm[2] | gm[3]))) {
        if (have && MODE == kContrib) a.partial[pos] = 0.0;
        if (have && MODE == kGrad) {
          double4* rec = reinterpret_cast<double4*>(a.partial + (int64_t)pos * 8);
          rec[0] = make_double4(0, 0, 0, 0);
          rec[1] = make_double4(0, 0, 0, 0);
        }
        continue;
      }
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
        WPROF(3);
        uint64_t lm[4];
#pragma unroll
        for (int w = 0; w < 4; ++w)
          lm[w] = gm[w] & ((uint64_t)alive_bits[2 * w] | ((uint64_t)alive_bits[2 * w + 1] << 32));
        // ---- P1: per-ray counts of the members in [j0, j1), flat offsets.
        //      Common case: everything left in the chunk fits the flat array
        //      (j1 = nG, one scan); otherwise the chunk is cut by Gaussians.
        int cnt_r = 0;
        uint32_t pre_lo = 0, pre_hi = 0;
        auto ray_counts = [&](int jb) {
          cnt_r = 0;
          pre_lo = pre_hi = 0;
          if (alive) {
#pragma unroll
            for (int w = 0; w < 8; ++w) {
              const int c = __popc(rows[w * kRays + tid] & range_mask(w, j0, jb));
              if (w < 4) pre_lo |= (uint32_t)cnt_r << (8 * w);
              else pre_hi |= (uint32_t)cnt_r << (8 * (w - 4));
              cnt_r += c;
            }
          }
        };
        int j1 = nG;
        ray_counts(j1);
        int total;
        int roff = block_scan(cnt_r, scan_tmp, total);
        if (total == 0) break;  // no live pair left in this chunk
        if (total > kCap) {     // block-uniform
          const int cnt_g = (have && tid >= j0)
                                ? __popcll(lm[0]) + __popcll(lm[1]) + __popcll(lm[2]) + __popcll(lm[3])
                                : 0;
          int tot_g;
          const int excl_g = block_scan(cnt_g, scan_tmp, tot_g);
          if (tid == j0) base_s = excl_g;
          __syncthreads();
          const bool fits = have && tid >= j0 && (excl_g + cnt_g - base_s) <= kCap;
          j1 = j0 + __syncthreads_count(fits);
          ray_counts(j1);
          roff = block_scan(cnt_r, scan_tmp, total);
        }
        WPROF(4);
        wpre[tid] = pre_lo;
        wpre[kRays + tid] = pre_hi;
        ray_off[tid] = roff;
        // replay space for this sub-chunk: the atomic's round trip overlaps P2/P3
        unsigned long long rp_o = 0;
        if (record && tid == 0) rp_o = atomicAdd(a.rp.cursor, (unsigned long long)total);
        __syncthreads();
        WPROF(5);
#if SDGR_WALK_P3_SCAN
        s_S0[tid] = S;
#endif
        // ---- P2: weights into the flat slots.  The warp's (Gaussian, ray)
        //      members go through a member list so every lane evaluates one
        //      exp per round whatever the per-Gaussian member counts.
        const bool mine = have && tid >= j0 && tid < j1;
        const int jw = tid >> 5;
        const uint32_t rmask_w = range_mask(jw, j0, j1);
        const uint32_t below = ((1u << lane) - 1u) & rmask_w;
        const uint32_t pshift = 8 * (jw & 3);
        const uint32_t* wp = wpre + (jw < 4 ? 0 : kRays);
        if (mine) {   // thread j: its own live member cells
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            uint64_t x = lm[w];
            while (x) {
              const int r = w * 64 + __ffsll((long long)x) - 1;
              x &= x - 1;
              const int p = ray_off[r] + (int)((wp[r] >> pshift) & 255u) + __popc(rows[jw * kRays + r] & below);
#if !SDGR_WALK_P2_FLAT
              const double dx = dsub((double)(tx * kTile + (r & 15)), su[tid]);
              const double dy = dsub((double)(ty * kTile + (r >> 4)), sv[tid]);
              const double wgt = exp(-quadform(sa0[tid], sa1[tid], sa2[tid], dx, dy));
              fw[p] = wgt;
              fs[p] = dmul(sk[tid], wgt);
#endif
              fj[p] = (uint8_t)tid;
              fr[p] = (uint8_t)r;
            }
          }
        }
        __syncthreads();
#if SDGR_WALK_P2_FLAT
        // the weights pair-parallel over the flat slots (<= kCap / 256 per
        // thread, whatever the per-Gaussian member counts)
        for (int p = tid; p < total; p += kRays) {
          const int j = fj[p], r = fr[p];
          const double dx = dsub((double)(tx * kTile + (r & 15)), su[j]);
          const double dy = dsub((double)(ty * kTile + (r >> 4)), sv[j]);
          const double wgt = exp(-quadform(sa0[j], sa1[j], sa2[j], dx, dy));
          fw[p] = wgt;
          fs[p] = dmul(sk[j], wgt);
        }
        __syncthreads();
#endif
        WPROF(6);
        // ---- P3: ray-serial log-transmittance prefix (additions only); the
        //      tau loads are issued 4 ahead of the dependent add chain
#if SDGR_WALK_P3_SCAN
        // balanced variant: a block segmented scan over the ray runs of the
        // flat array (<= kCap / 256 consecutive entries per thread), S at a
        // pair = the ray's S at the sub-chunk start + the run's exclusive sum
        {
          constexpr int kE = (kCap + kRays - 1) / kRays;
          const double kInf = __longlong_as_double(0x7ff0000000000000ll);
          const int E = (total + kRays - 1) / kRays;
          const int q0 = E * tid;
          const int cnt = max(0, min(E, total - q0));
          double v[kE], tq[kE];
          bool hd[kE];
#pragma unroll
          for (int e = 0; e < kE; ++e) {
            v[e] = 0.0;
            tq[e] = 0.0;
            hd[e] = true;
            if (e < cnt) {
              const int q = q0 + e;
              tq[e] = fs[q];
              v[e] = tq[e];
              hd[e] = q == 0 || fr[q - 1] != fr[q];
            }
          }
          block_seg_scan8<kE>(v, hd, cnt, s_agg8, s_flag8);
#pragma unroll
          for (int e = 0; e < kE; ++e) {
            if (e < cnt) {
              const int q = q0 + e, r = fr[q];
              const double S0 = s_S0[r];
              const double Sx = dadd(S0, dsub(v[e], tq[e]));
              fs[q] = Sx < a.s_stop ? Sx : kInf;  // dead: T = 0
              if (q == total - 1 || fr[q + 1] != r) s_S1[r] = dadd(S0, v[e]);
            }
          }
        }
        if (false) {
#else
        if (cnt_r > 0) {
#endif
          const double kInf = __longlong_as_double(0x7ff0000000000000ll);
          const int p1 = roff + cnt_r;
          int p = roff;
          while (p < p1 && S < a.s_stop) {
            double t4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) t4[k] = p + k < p1 ? fs[p + k] : 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              if (p + k < p1) {
                const bool live = S < a.s_stop;
                fs[p + k] = live ? S : kInf;  // dead: T = 0
                if (live) S = dadd(S, t4[k]);
              }
            }
            p += 4;
          }
          for (; p < p1; ++p) fs[p] = kInf;
          alive = S < a.s_stop;
        }
#ifdef SDGR_WALK_PROFILE
        __syncthreads();
        WPROF(10);
#endif
        if (record && tid == 0) {
          const unsigned long long o = rp_o;
          const bool fits = o + (unsigned long long)total <= (unsigned long long)a.rp.capacity &&
                            n_desc < a.rp.desc_per_item;
          rp_off = fits ? (long long)o : -1ll;
          if (fits) {
            int4 d;
            d.x = (int)o; d.y = total; d.z = cs; d.w = j0 | (j1 << 16);
            reinterpret_cast<int4*>(a.rp.desc)[(int64_t)item * a.rp.desc_per_item + n_desc] = d;
          } else {
            a.rp.cursor[1] = 1ull;  // overflow: the host must re-walk
          }
        }
        __syncthreads();
        WPROF(7);
#if SDGR_WALK_P3_SCAN
        if (cnt_r > 0) {
          S = s_S1[tid];
          alive = S < a.s_stop;
        }
#endif
        // ---- P4: flat pair-parallel transmittance and contributions
        const long long lo = record ? rp_off : -1ll;
        if (lo >= 0) ++n_desc;  // count only descriptors actually written (log overflow)
        for (int p = tid; p < total; p += kRays) {
          const int j = fj[p];
          const double wgt = fw[p];
          const double tau = sk[j] * wgt;
          const double T = exp(-fs[p]);
          const double em1 = expm1(-tau);
          const double oma = -em1;
          if (lo >= 0) {
            // the backward needs only these per live pair: no transcendentals there
            a.rp.y1[lo + p] = T * oma;
            a.rp.t2[lo + p] = T * (1.0 + em1);  // T e^-tau
            a.rp.w[lo + p] = wgt;
            a.rp.j[lo + p] = (uint8_t)j;
            a.rp.r[lo + p] = fr[p];
          }
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
        WPROF(8);
        // ---- P5: ray-serial sums of g*contrib (backward)
        if (MODE == kGSum) {
          for (int p = roff; p < roff + cnt_r; ++p) accd += fs[p];
        } else if (MODE == kGrad) {
          for (int p = roff; p < roff + cnt_r; ++p) {
            rem -= fs[p];
            fs[p] = rem;  // downstream sum after this pair
          }
          __syncthreads();
        }
        // ---- P7: Gaussian-parallel reduction in cell order
        if (MODE != kGSum && mine) {
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
        __syncthreads();
        WPROF(9);
        j0 = j1;
      }
      if (MODE == kContrib && have) a.partial[pos] = racc[0];
      if (MODE == kGrad && have) {
        double4* rec = reinterpret_cast<double4*>(a.partial + (int64_t)pos * 8);
        rec[0] = make_double4(racc[0] * sg[tid], racc[1], racc[2], racc[3]);
        rec[1] = make_double4(racc[4], racc[5], racc[6], 0.0);
      }
    }
    if (SDGR_WALK_BULK && pending) {   // a prefetch the early exit left in flight
      mbar_wait(&s_mbar, parity);
      parity ^= 1u;
    }
    // every Gaussian of the segment owns a record: zero the ones past an early exit
    if (MODE != kGSum) {
      for (int i = cs + tid; i < end; i += kChunk) {
        const int p = a.rec[i].pos;
        if (MODE == kContrib) a.partial[p] = 0.0;
        else {
          double4* rec = reinterpret_cast<double4*>(a.partial + (int64_t)p * 8);
          rec[0] = make_double4(0, 0, 0, 0);
          rec[1] = make_double4(0, 0, 0, 0);
        }
      }
    }
    if (MODE == kGSum) a.seg_out[slot_ray] = accd;
    if (MODE == kContrib && a.seg_out) a.seg_out[slot_ray] = S;  // first segment: S after it
    if (record && tid == 0) a.rp.desc_count[item] = min(n_desc, a.rp.desc_per_item);
    if (MODE == kContrib && __syncthreads_or(bad) && tid == 0) atomicOr(a.status + SDGR_STATUS_NONFINITE, 1);
  }
}

// ============================================================ replay ==========
// Backward over the live-pair log the forward walk wrote: per work item, its
// sub-chunk descriptors in walk order; per descriptor the live pairs in
// ray-major, depth-minor order with y1 = T(1 - e^-tau), t2 = T e^-tau and w
// (the forward already evaluated every transcendental the backward needs).  No binning, membership
// or weight work is repeated, and only live pairs are touched.
//   kGSum: per (item, ray) sum of g * contrib          (backward.py:129-139)
//   kGrad: reverse-recurrence terms, reduced per Gaussian in ray order into
//          one partial record per (tile, Gaussian)      (backward.py:122-148)
struct ReplayArgs {
  sdgr_replay rp;
  const sdgr_pair_rec* rec;
  const int32_t* items;
  const int32_t* n_items;
  uint32_t* counter;
  int tiles_x;
  const double* gvec;     // dL/dI
  const double* seg_g;    // kGrad
  const double* seg_d;    // kGrad
  double* seg_out;        // kGSum
  double* partial;        // kGrad: (n_pairs, 8), every record written
};

template <int MODE, bool kBig>
struct ReplayCfg {
  // fY (+ fW, fD) doubles, fj, fr bytes (+ perm u16)
  static constexpr size_t kSmem = (size_t)replay_cap<kBig>() * (MODE == kGrad ? 3 * 8 + 2 + 2 : 8 + 2);
};

// Per descriptor (<= kReplayCap log entries of Gaussians [j0, j1) of one chunk):
//   L  stage the Gaussians and the entries;
//   B  entry-parallel g*contrib (ceil(n/256) contiguous entries per thread), a block
//      segmented scan over the ray runs: per-ray sums (kGSum) or the downstream
//      sum D after each pair (kGrad) -- no ray-serial loops;
//   C  kGrad: counting sort of the entries into Gaussian-major order (ray
//      bitmaps per Gaussian), then thread j sums Gaussian j's gradient terms
//      over its entries in ray order: one partial record per (tile, Gaussian)
//      pair, written once.  (A warp-balanced variant -- up to 8 contiguous
//      entries per lane, warp segmented scan of the 7-term vectors -- held 28
//      doubles live: 126 registers, 2 CTAs/SM, 7.47 vs 6.49 ms/step.)  Pairs
//      of the item no descriptor covers get zero records here, so partial_g
//      needs no memset.
template <int MODE, bool kBig>
__global__ void __launch_bounds__(256, MODE == kGrad ? (kBig ? 3 : SDGR_MINB_REPLAY_GRAD)
                                                     : (kBig ? SDGR_MINB_REPLAY_GSUM_BIG : SDGR_MINB_REPLAY_GSUM)) k_replay(ReplayArgs a) {
  constexpr bool kG = MODE == kGrad;
  constexpr int kCap = replay_cap<kBig>();
  __shared__ double sk[kChunk], sp[kChunk], sg[kChunk];
  __shared__ double su[kG ? kChunk : 1], sv[kG ? kChunk : 1], sa0[kG ? kChunk : 1], sa1[kG ? kChunk : 1],
      sa2[kG ? kChunk : 1];
  __shared__ int32_t spos[kG ? kChunk : 1];
  __shared__ double ray_acc[kRays];                 // kGSum: per-ray sum; kGrad: remaining sum per ray
  __shared__ uint32_t jm[kG ? 8 * kChunk : 1];      // jm[w*256 + j]: rays of Gaussian j (bit r&31 of word r>>5)
  __shared__ uint32_t jpre[kG ? 2 * kChunk : 1];    // per Gaussian: byte prefix counts of its jm words
  __shared__ int32_t gstart[kG ? kChunk + 1 : 1];
  __shared__ double s_agg[8];
  __shared__ int s_flag[8];
  __shared__ int32_t scan_tmp[8];
  __shared__ int item_s;
  __shared__ int4 s_desc[kDescCache];               // the item's first descriptors
  extern __shared__ double dyn[];
  double* fY = dyn;                                  // y1 = T (1 - e^-tau)
  double* fW = fY + kCap;                            // kGrad: w
  double* fD = fW + (kG ? kCap : 0);                 // kGrad: x - D (x = g T e^-tau P, D downstream sum)
  uint16_t* perm = reinterpret_cast<uint16_t*>(fD + (kG ? kCap : 0));  // kGrad: Gaussian-major -> log
  uint8_t* fj = reinterpret_cast<uint8_t*>(perm + (kG ? kCap : 0));
  uint8_t* fr = fj + kCap;
  const int tid = threadIdx.x;
  const int n_items = *a.n_items;
  while (true) {
    __syncthreads();
    if (tid == 0) item_s = (int)atomicAdd(a.counter, 1u);
    __syncthreads();
    if (item_s >= n_items) return;
    const int item = SDGR_ORDER_REPLAY ? a.items[4 * item_s + 3] : item_s;   // processing order (k_make_items)
    // item metadata, its descriptors and the per-ray seeds load in parallel
    const int4 it = reinterpret_cast<const int4*>(a.items)[item];
    const int nd = a.rp.desc_count[item];
    const int4* descs = reinterpret_cast<const int4*>(a.rp.desc) + (int64_t)item * a.rp.desc_per_item;
    if (tid < min(nd, kDescCache)) s_desc[tid] = descs[tid];
    const int tx = it.x % a.tiles_x, ty = it.x / a.tiles_x;
    const int64_t slot_ray = (int64_t)item * kRays + tid;
    ray_acc[tid] = kG ? a.seg_d[slot_ray] + a.seg_g[slot_ray] : 0.0;
    int covered = it.y;  // kGrad: pairs below this have a record
    for (int k = 0; k < nd; ++k) {
      __syncthreads();
      const int4 d = k < kDescCache ? s_desc[k] : descs[k];
      const int64_t off = d.x;
      const int n = d.y, cs = d.z, j0 = d.w & 0xffff, j1 = d.w >> 16;
      // ---- L: Gaussians and entries
      if (kG) {
        for (int i = covered + tid; i < cs + j0; i += kRays) {
          double4* rp = reinterpret_cast<double4*>(a.partial + (int64_t)__ldg(&a.rec[i].pos) * 8);
          rp[0] = make_double4(0, 0, 0, 0);
          rp[1] = make_double4(0, 0, 0, 0);
        }
        covered = cs + j1;
#pragma unroll
        for (int w = 0; w < 8; ++w) jm[w * kChunk + tid] = 0u;
      }
      // this thread's Gaussian (kGSum: only P and the scene index; kGrad: the
      // record) and its first two log rows are loaded before either is
      // consumed, so their latencies -- and kGSum's dependent dL/dI gather --
      // overlap
      const bool mine = tid >= j0 && tid < j1;
      sdgr_pair_rec r{};
      double ph = 0.0;
      int prim = 0;
      if (mine) {
        if (kG) {
          r = load_rec(a.rec + cs + tid);
        } else {
          ph = __ldg(&a.rec[cs + tid].phase);
          prim = __ldg(&a.rec[cs + tid].prim);
        }
      }
      auto load_rows = [&](int p, double& y_a, double& y_b, double& w_a, double& w_b, double& t_a, double& t_b,
                           uint8_t& j_a, uint8_t& j_b, uint8_t& r_a, uint8_t& r_b) {
        const int p2 = p + kRays;
        const bool one = p < n, two = p2 < n;
        y_a = one ? a.rp.y1[off + p] : 0.0;
        y_b = two ? a.rp.y1[off + p2] : 0.0;
        if (kG) {
          w_a = one ? a.rp.w[off + p] : 0.0;
          t_a = one ? a.rp.t2[off + p] : 0.0;
          w_b = two ? a.rp.w[off + p2] : 0.0;
          t_b = two ? a.rp.t2[off + p2] : 0.0;
        }
        j_a = one ? a.rp.j[off + p] : 0; r_a = one ? a.rp.r[off + p] : 0;
        j_b = two ? a.rp.j[off + p2] : 0; r_b = two ? a.rp.r[off + p2] : 0;
      };
      auto store_rows = [&](int p, double y_a, double y_b, double w_a, double w_b, double t_a, double t_b,
                            uint8_t j_a, uint8_t j_b, uint8_t r_a, uint8_t r_b) {
        const int p2 = p + kRays;
        if (p < n) {
          fY[p] = y_a; fj[p] = j_a; fr[p] = r_a;
          if (kG) { fW[p] = w_a; fD[p] = t_a; }
        }
        if (p2 < n) {
          fY[p2] = y_b; fj[p2] = j_b; fr[p2] = r_b;
          if (kG) { fW[p2] = w_b; fD[p2] = t_b; }
        }
      };
      // log entries: two rows of loads in flight per thread; kGrad also
      // stages t2 here (into fD) so stage B reads no global memory
      double y_a = 0, y_b = 0, w_a = 0, w_b = 0, t_a = 0, t_b = 0;
      uint8_t j_a = 0, j_b = 0, r_a = 0, r_b = 0;
      load_rows(tid, y_a, y_b, w_a, w_b, t_a, t_b, j_a, j_b, r_a, r_b);
      if (mine) {
        if (kG) {
          sk[tid] = r.kappa;
          sp[tid] = r.phase;
          sg[tid] = a.rp.gpair[cs + tid];  // written by the kGSum pass: no prim -> dL/dI gather chain
          su[tid] = r.u; sv[tid] = r.v;
          sa0[tid] = r.a00; sa1[tid] = r.a01; sa2[tid] = r.a11;
          spos[tid] = r.pos;
        } else {
          const double g = a.gvec[prim];
          sp[tid] = ph;
          sg[tid] = g;
          a.rp.gpair[cs + tid] = g;
        }
      }
      store_rows(tid, y_a, y_b, w_a, w_b, t_a, t_b, j_a, j_b, r_a, r_b);
      for (int p = tid + 2 * kRays; p < n; p += 2 * kRays) {
        load_rows(p, y_a, y_b, w_a, w_b, t_a, t_b, j_a, j_b, r_a, r_b);
        store_rows(p, y_a, y_b, w_a, w_b, t_a, t_b, j_a, j_b, r_a, r_b);
      }
      __syncthreads();
      // ---- B: g*contrib per entry, segmented scan over the ray runs
      // E contiguous entries per thread, E = ceil(n / 256) <= 8: all threads share the work
      const int E = (n + kRays - 1) / kRays;
      const int q0 = E * tid;
      const int cnt = max(0, min(E, n - q0));
      constexpr int kE = kCap / kRays;   // entries per thread at most: 4 (small config) or 8
      double v[kE];
      bool hd[kE];
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        v[e] = 0.0;
        hd[e] = true;
        if (e < cnt) {
          const int q = q0 + e;
          const int j = fj[q], r = fr[q];
          v[e] = sg[j] * (fY[q] * sp[j]);
          if (kG) fD[q] = sg[j] * fD[q] * sp[j];  // x (fD held t2), thread-private until P7
          hd[e] = q == 0 || fr[q - 1] != r;
          if (kG) atomicOr(jm + (r >> 5) * kChunk + j, 1u << (r & 31));
        }
      }
      block_seg_scan8(v, hd, cnt, s_agg, s_flag);
      if (kG) {
#pragma unroll
        for (int e = 0; e < kE; ++e)
          if (e < cnt) fD[q0 + e] -= ray_acc[fr[q0 + e]] - v[e];
        __syncthreads();
      }
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        const int q = q0 + e;
        if (e < cnt && (q == n - 1 || fr[q + 1] != fr[q])) {
          if (kG) ray_acc[fr[q]] -= v[e];
          else ray_acc[fr[q]] += v[e];
        }
      }
      if (!kG) continue;
      // ---- C: Gaussian-major order
      {
        int c = 0;
        uint32_t plo = 0, phi = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          if (w < 4) plo |= (uint32_t)c << (8 * w);
          else phi |= (uint32_t)c << (8 * (w - 4));
          c += __popc(jm[w * kChunk + tid]);
        }
        jpre[tid] = plo;
        jpre[kChunk + tid] = phi;
        int tot;
        const int gs = block_scan(c, scan_tmp, tot);
        gstart[tid] = gs;
        if (tid == 0) gstart[kChunk] = tot;
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        if (e < cnt) {
          const int q = q0 + e;
          const int j = fj[q], r = fr[q], w = r >> 5;
          const int rank = (int)((jpre[(w < 4 ? 0 : kChunk) + j] >> (8 * (w & 3))) & 255u) +
                           __popc(jm[w * kChunk + j] & ((1u << (r & 31)) - 1u));
          perm[gstart[j] + rank] = (uint16_t)q;
        }
      }
      __syncthreads();
      // C': thread j sums its own entries serially, in ray order (Gaussian-
      // major via perm): one partial record per (tile, Gaussian)
      if (tid >= j0 && tid < j1) {
        double acc[7] = {0, 0, 0, 0, 0, 0, 0};
        const int lo = gstart[tid], hi = gstart[tid + 1];
#pragma unroll 1   // no unrolled body + remainder split over the per-Gaussian entry counts (kGrad -1.3 %)
        for (int qq = lo; qq < hi; ++qq) {
          const int p = perm[qq];
          const int r = fr[p];
          const double dx = dsub((double)(tx * kTile + (r & 15)), su[tid]);
          const double dy = dsub((double)(ty * kTile + (r >> 4)), sv[tid]);
          grad_terms(fY[p], fD[p] * fW[p], sk[tid], dx, dy, sa0[tid], sa1[tid], sa2[tid], acc);
        }
        double4* rp = reinterpret_cast<double4*>(a.partial + (int64_t)spos[tid] * 8);
        rp[0] = make_double4(acc[0] * sg[tid], acc[1], acc[2], acc[3]);
        rp[1] = make_double4(acc[4], acc[5], acc[6], 0.0);
      }
    }

    if (kG) {
      // pairs after the last descriptor
      for (int i = covered + tid; i < it.z; i += kRays) {
        double4* rp = reinterpret_cast<double4*>(a.partial + (int64_t)__ldg(&a.rec[i].pos) * 8);
        rp[0] = make_double4(0, 0, 0, 0);
        rp[1] = make_double4(0, 0, 0, 0);
      }
    } else {
      __syncthreads();
      a.seg_out[slot_ray] = ray_acc[tid];
    }
  }
}

// Per-ray exclusive prefix (forward) or suffix (backward) over a tile's
// segment items.  One CTA per tile, thread = ray.
template <bool kSuffix, bool kFixIn = false>
__global__ void __launch_bounds__(256) k_seg_scan(const int32_t* __restrict__ range,
                                                  const int32_t* __restrict__ tile_first, int seg_len,
                                                  const double* __restrict__ in, double* __restrict__ out) {
  const int t = blockIdx.x;
  const int cnt = range[2 * t + 1] - range[2 * t];
  const int nseg = (cnt + seg_len - 1) / seg_len;
  if (nseg == 0) return;
  const int64_t first = tile_first[t];
  double run = 0.0;
  // loads of 8 segments are issued before the dependent adds
  for (int k0 = 0; k0 < nseg; k0 += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u;
      v[u] = 0.0;
      if (k < nseg) {
        const int64_t s = (first + (kSuffix ? nseg - 1 - k : k)) * kRays + threadIdx.x;
        v[u] = kFixIn ? (double)reinterpret_cast<const unsigned long long*>(in)[s] * kFixInv : in[s];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u;
      if (k < nseg) {
        out[(first + (kSuffix ? nseg - 1 - k : k)) * kRays + threadIdx.x] = run;
        run += v[u];
      }
    }
  }
}

// intensity[g] = sum of its per-tile partials, in pre-sort (tile-id) order.
__global__ void __launch_bounds__(256) k_reduce_intensity(const int32_t* pair_start, const int32_t* n_tiles,
                                                          const double* partial, int64_t n, int64_t cap,
                                                          double* out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  const int s = pair_start[g];
  const int64_t room = cap - s > 0 ? cap - s : 0;   // capacity overflow: stay in bounds
  const int c = n_tiles[g] < room ? n_tiles[g] : (int)room;
  double acc = 0.0;
  for (int k = 0; k < c; ++k) acc += partial[s + k];
  out[g] = acc;
}


template <int MODE, bool kBig>
static int walk_grid(int max_items) {
  static int per_sm = 0;
  if (per_sm == 0) {
    const size_t smem = WalkCfg<MODE, kBig>::kSmem;
    cudaFuncSetAttribute(k_walk<MODE, kBig>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_walk<MODE, kBig>, 256, smem);
    per_sm = b > 0 ? b : 1;
  }
  return max(1, min(max_items, persistent_grid(per_sm)));
}

template <int MODE, bool kBig>
static int launch_walk_cfg(const WalkArgs& a, int max_items, cudaStream_t st) {
  if (cudaMemsetAsync(a.counter, 0, sizeof(uint32_t), st) != cudaSuccess) return SDGR_ERR_CUDA;
  {
    KernelTimer kt(MODE == kContrib ? SDGR_K_WALK : 0, st);
    k_walk<MODE, kBig><<<walk_grid<MODE, kBig>(max_items), 256, WalkCfg<MODE, kBig>::kSmem, st>>>(a);
  }
  note_launch();
  return check_launch();
}

template <int MODE>
static int launch_walk(const WalkArgs& a, const sdgr_tiles& t, cudaStream_t st) {
  return big_walk(t) ? launch_walk_cfg<MODE, true>(a, t.max_items, st)
                     : launch_walk_cfg<MODE, false>(a, t.max_items, st);
}

static WalkArgs base_args(const sdgr_view& v, const sdgr_tiles& t) {
  WalkArgs a{};
  a.n_cols = v.n_u;
  a.n_rows = v.n_v;
  a.tiles_x = t.tiles_x;
  a.cutoff = v.cutoff;
  a.rec = t.pair_rec;
  a.items = t.items;
  a.n_items = t.n_items;
  a.counter = reinterpret_cast<uint32_t*>(t.n_items + 2);
  return a;
}

int launch_composite_forward(const sdgr_view& v, const sdgr_projection& p, const sdgr_tiles& t,
                             double s_stop, double* seg_sum, double* seg_base, double* partial_I,
                             double* intensity, int32_t* status, const sdgr_replay* rp, cudaStream_t st) {
  if (rp && cudaMemsetAsync(rp->cursor, 0, sizeof(unsigned long long), st) != cudaSuccess)  // [1] is sticky
    return SDGR_ERR_CUDA;
  if (t.n_pairs > 0) {
    // Pass A: per-(segment, ray) optical depth, then the per-ray exclusive
    // prefix over the tile's segments, then the walk.  (A two-phase variant
    // -- first segments walked exactly, pass A only on rays still alive --
    // measured slower: the first phase runs at one CTA per tile.)
    uint32_t* counter = reinterpret_cast<uint32_t*>(t.n_items + 2);
    // seg_sum is reused as u64 fixed-point counters (same 8-byte slots).
    unsigned long long* seg_fx = reinterpret_cast<unsigned long long*>(seg_sum);
    if (cudaMemsetAsync(counter, 0, sizeof(uint32_t), st) != cudaSuccess) return SDGR_ERR_CUDA;
    if (cudaMemsetAsync(seg_fx, 0, (size_t)t.max_items * kRays * sizeof(unsigned long long), st) != cudaSuccess)
      return SDGR_ERR_CUDA;
    static int per_sm = 0;
    if (per_sm == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_segsum, 256, 0);
    {
      KernelTimer kt(SDGR_K_SEGSUM, st);
      k_segsum<<<max(1, min(t.max_items, persistent_grid(per_sm))), 256, 0, st>>>(
          t.pair_rec, t.items, t.n_items, counter, t.tiles_x, v.cutoff, seg_fx);
    }
    k_seg_scan<false, true><<<t.n_tiles, 256, 0, st>>>(t.tile_range, t.tile_first, t.seg_len, seg_sum, seg_base);
    note_launch(2);
    WalkArgs a = base_args(v, t);
    a.s_stop = s_stop;
    a.seg_base = seg_base;
    a.partial = partial_I;
    a.status = status;
    if (rp) a.rp = *rp;
    const int rc = launch_walk<kContrib>(a, t, st);
    if (rc) return rc;
  }
  k_reduce_intensity<<<(unsigned)((p.n + 255) / 256), 256, 0, st>>>(t.pair_start, p.comp.n_tiles, partial_I,
                                                                     p.n, t.n_pairs, intensity);
  note_launch();
  return check_launch();
}

// image: (n_rg, n_az) FP64; part: scratch of >= n_rg*n_az + 1 u64 (8-byte)
// slots (the pixel sums, then the view's max intensity).
int launch_splat(const sdgr_view& v, const sdgr_projection& p, const double* intensity, double* part,
                 double* image, cudaStream_t st) {
  const int64_t npix = (int64_t)v.n_az * v.n_rg;
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(part);
  if (cudaMemsetAsync(acc, 0, sizeof(unsigned long long) * (npix + 1), st) != cudaSuccess) return SDGR_ERR_CUDA;
  const unsigned gb = (unsigned)((p.n + 255) / 256);
  k_max_intensity<<<std::min<unsigned>(gb, 2u * (unsigned)sm_count()), 256, 0, st>>>(p.flags, intensity, p.n,
                                                                                     acc + npix);
  {
    const int64_t ng = (p.n + 31) / 32;
    int64_t wperm = std::max<int64_t>(1, (int64_t)(0.6180339887 * (double)ng));
    while (std::gcd(wperm, ng) != 1) ++wperm;
    KernelTimer kt(SDGR_K_SPLAT, st);
    k_splat<<<(unsigned)std::max<int64_t>(1, (ng + 7) / 8), 256, 0, st>>>(v, p.img, p.flags, intensity, p.n, wperm, acc, acc + npix);
  }
  k_splat_finish<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(acc, npix, image);
  note_launch(3);
  return check_launch();
}

template <bool kBig>
static int launch_replay(ReplayArgs& r, const sdgr_tiles& t, double* seg_g, double* seg_d, double* partial_g,
                         cudaStream_t st) {
  static int per_sm[2] = {0, 0};
  if (per_sm[0] == 0) {
    cudaFuncSetAttribute(k_replay<kGSum, kBig>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)ReplayCfg<kGSum, kBig>::kSmem);
    cudaFuncSetAttribute(k_replay<kGrad, kBig>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)ReplayCfg<kGrad, kBig>::kSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], k_replay<kGSum, kBig>, 256,
                                                  ReplayCfg<kGSum, kBig>::kSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], k_replay<kGrad, kBig>, 256,
                                                  ReplayCfg<kGrad, kBig>::kSmem);
  }
  if (cudaMemsetAsync(r.counter, 0, sizeof(uint32_t), st) != cudaSuccess) return SDGR_ERR_CUDA;
  {
    KernelTimer kt(SDGR_K_REPLAY_GSUM, st);
    k_replay<kGSum, kBig><<<max(1, min(t.max_items, persistent_grid(per_sm[0]))), 256,
                            ReplayCfg<kGSum, kBig>::kSmem, st>>>(r);
  }
  k_seg_scan<true><<<t.n_tiles, 256, 0, st>>>(t.tile_range, t.tile_first, t.seg_len, seg_g, seg_d);
  note_launch(2);
  // k_replay<kGrad> writes every pair's record (zeros for pairs it skips)
  if (cudaMemsetAsync(r.counter, 0, sizeof(uint32_t), st) != cudaSuccess) return SDGR_ERR_CUDA;
  r.seg_out = nullptr;
  r.seg_g = seg_g;
  r.seg_d = seg_d;
  r.partial = partial_g;
  {
    KernelTimer kt(SDGR_K_REPLAY_GRAD, st);
    k_replay<kGrad, kBig><<<max(1, min(t.max_items, persistent_grid(per_sm[1]))), 256,
                            ReplayCfg<kGrad, kBig>::kSmem, st>>>(r);
  }
  note_launch();
  return check_launch();
}

int launch_grad_intensity(const sdgr_view& v, const sdgr_projection& p, const sdgr_tiles& t,
                          double s_stop, const double* seg_base, const double* dL_dI, double* seg_g,
                          double* seg_d, double* partial_g, const sdgr_replay* rp, cudaStream_t st) {
  if (t.n_pairs == 0) return SDGR_OK;
  if (rp) {
    // replay the forward's live-pair log
    ReplayArgs r{};
    r.rp = *rp;
    r.rec = t.pair_rec;
    r.items = t.items;
    r.n_items = t.n_items;
    r.counter = reinterpret_cast<uint32_t*>(t.n_items + 2);
    r.tiles_x = t.tiles_x;
    r.gvec = dL_dI;
    r.seg_out = seg_g;
    return big_walk(t) ? launch_replay<true>(r, t, seg_g, seg_d, partial_g, st)
                       : launch_replay<false>(r, t, seg_g, seg_d, partial_g, st);
  }
  WalkArgs a = base_args(v, t);
  a.s_stop = s_stop;
  a.seg_base = seg_base;
  a.gvec = dL_dI;
  a.seg_out = seg_g;
  int rc = launch_walk<kGSum>(a, t, st);
  if (rc) return rc;
  k_seg_scan<true><<<t.n_tiles, 256, 0, st>>>(t.tile_range, t.tile_first, t.seg_len, seg_g, seg_d);
  note_launch();
  a.seg_out = nullptr;
  a.seg_g = seg_g;
  a.seg_d = seg_d;
  a.partial = partial_g;
  return launch_walk<kGrad>(a, t, st);
}

}  // namespace sdgr

#ifdef SDGR_WALK_PROFILE
extern "C" int sdgr_debug_walk_profile(unsigned long long* out) {
  if (cudaMemcpyFromSymbol(out, sdgr::g_walk_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 4;
  unsigned long long z[16] = {};
  return cudaMemcpyToSymbol(sdgr::g_walk_prof, z, sizeof(z)) == cudaSuccess ? 0 : 4;
}
#endif
