// common.cuh — shared device helpers for the SDGR sm_100a kernels.
//
// The FP64 "key chain" (everything that decides which (cell, Gaussian) pairs
// exist and in which order) is written with explicit round-to-nearest
// intrinsics so nvcc can neither contract nor reassociate it.  The op order
// follows the reference exactly as measured on its host:
//   x_r = fma(p2, R2, fma(p1, R1, p0*R0)) + T   (OpenBLAS dgemm, geometry.py:249)
//   Sigma = M M^T with the same FMA chain         (scene.py:96)
//   mc Sigma mc^T summed sequentially over (b,c)  (np.einsum, geometry.py:271)
// and is mirrored bit-for-bit by the C oracle (oracle/keychain.c).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sdgr.h"

namespace sdgr {

constexpr int kTile = SDGR_TILE;        // 16
constexpr int kRays = SDGR_TILE_RAYS;   // 256 rays (cells) per tile
constexpr int kChunk = 256;             // Gaussians staged per tile-walk chunk

// Minimum resident 256-thread blocks per SM for the Gaussian-parallel FP64
// kernels.  k_grad_image: 64 registers (4 blocks) hides the FP64 dependency
// latency better than the few spills it costs (2.57 -> 2.42 ms/step on the
// c4 bench; 5 and 6 were slower).  k_project: 3 blocks, 80 registers and no
// spills since the structural-zero sandwich (4.33 -> 4.14 ms/step, +0.6 %
// views/s over 4; round 1 measured 4 better).  Overridable for A/B builds
// via SDGR_EXTRA_FLAGS.
#ifndef SDGR_MINB_PROJECT
#define SDGR_MINB_PROJECT 3
#endif
#ifndef SDGR_MINB_REPLAY_GSUM
#define SDGR_MINB_REPLAY_GSUM 6   // 40 registers: +0.6 % views/s in the concurrent step (c4)
#endif
#ifndef SDGR_MINB_REPLAY_GRAD   // 4: 64 registers, no spills at the 1024-entry replay buffer
#define SDGR_MINB_REPLAY_GRAD 4
#endif
#ifndef SDGR_MINB_GEOMETRY
#define SDGR_MINB_GEOMETRY 5
#endif
#ifndef SDGR_MINB_GRAD_IMAGE
#define SDGR_MINB_GRAD_IMAGE 4
#endif

// ---- explicit-rounding FP64 helpers (no contraction) -----------------------
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

// ---- e^x for x <= 0 on the compositing path ---------------------------------
// Table-driven (Tang): x = (64 e + j) ln2/64 + r, |r| <= ln2/128, e^x =
// 2^e 2^(j/64) e^r with e^r - 1 a degree-5 polynomial (truncation < 0.2 ulp);
// <= 2 ulp against libdevice exp (tests/test_gpu_stages.py), deterministic,
// ~2/3 of libdevice's instructions (its degree-11 polynomial needs a 64-bit
// constant per term) but a dependent table load.  Used where it measured
// faster: the imaging-plane backward (k_grad_image 2.30 -> 2.20 ms/step)
// and the splat; pass A and the walk keep exp() (their exp feeds a short
// dependent chain and the table load made them slower: 4.14 -> 4.73 and
// 7.77 -> 7.90 ms/step).  Outside (-708, 0] (underflow, -inf, NaN) it
// defers to exp().
#ifndef SDGR_FAST_EXP
#define SDGR_FAST_EXP 1
#endif
static __device__ const double kExp2Tab[64] = {
  1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284,
  1.0442737824274138, 1.0556451783605572, 1.0671404006768237, 1.0787607977571199,
  1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418,
  1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812,
  1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687,
  1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783,
  1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303,
  1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112,
  1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647,
  1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384,
  1.5422108254079407, 1.559004400237837, 1.5759808451078865, 1.593142151342267,
  1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364,
  1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062,
  1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989,
  1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656,
  1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951};

__device__ __forceinline__ double nexp(double x) {
#if SDGR_FAST_EXP
  if (!(x > -708.0)) return exp(x);
  const double shifter = 6755399441055744.0;   // 1.5 * 2^52: round-to-integer in the low word
  const double ts = fma(x, 92.33248261689366, shifter);   // x * 64 / ln2
  const int k = __double2loint(ts);
  const double kd = ts - shifter;
  double r = fma(kd, -0.010830424696223417, x);           // ln2/64, 36 significant bits: kd * hi exact
  r = fma(kd, -2.572804622327669e-14, r);
  double p = fma(fma(fma(fma(r, 1.0 / 120.0, 1.0 / 24.0), r, 1.0 / 6.0), r, 0.5), r, 1.0);
  p *= r;                                                  // e^r - 1
  const double T = __ldg(kExp2Tab + (k & 63));
  const double y = fma(T, p, T);
  return __hiloint2double(__double2hiint(y) + ((k >> 6) << 20), __double2loint(y));
#else
  return exp(x);
#endif
}

// np.maximum(x, 0.0): NaN propagates (fmax would drop it).
__device__ __forceinline__ double np_max0(double x) { return (x >= 0.0 || x != x) ? x : 0.0; }

// Deterministic FP64 exp shared with the oracle (oracle/keychain.c:sdgr_exp).
// Cody-Waite reduction by ln2, degree-13 Taylor polynomial in Horner/FMA
// form, exact power-of-two scaling.  <= ~0.75 ulp; identical bits on host and
// device because every step is a single IEEE operation.
__device__ __forceinline__ double sdgr_exp(double x) {
  if (!(x == x)) return x;
  if (x > 709.782712893384) return __longlong_as_double(0x7ff0000000000000ll);
  if (x < -745.1332191019412) return 0.0;
  const double kInvLn2 = 1.4426950408889634;
  const double kLn2Hi = 6.93147180369123816490e-01;
  const double kLn2Lo = 1.90821492927058770002e-10;
  double n = rint(dmul(x, kInvLn2));
  double r = dfma(-n, kLn2Hi, x);
  r = dfma(-n, kLn2Lo, r);
  double p = 1.0 / 6227020800.0;          // 1/13!
  p = dfma(p, r, 1.0 / 479001600.0);      // 1/12!
  p = dfma(p, r, 1.0 / 39916800.0);
  p = dfma(p, r, 1.0 / 3628800.0);
  p = dfma(p, r, 1.0 / 362880.0);
  p = dfma(p, r, 1.0 / 40320.0);
  p = dfma(p, r, 1.0 / 5040.0);
  p = dfma(p, r, 1.0 / 720.0);
  p = dfma(p, r, 1.0 / 120.0);
  p = dfma(p, r, 1.0 / 24.0);
  p = dfma(p, r, 1.0 / 6.0);
  p = dfma(p, r, 0.5);
  double r2 = dmul(r, r);
  double t = dfma(r2, p, r);
  double e = dadd(1.0, t);
  return scalbn(e, (int)n);
}

// Order-preserving uint64 key of an FP64 depth (-0.0 canonicalised to +0.0 so
// that ties fall back to the index, as np.lexsort compares -0.0 == 0.0).
__device__ __forceinline__ uint64_t depth_key(double d) {
  if (d == 0.0) d = 0.0;
  uint64_t b = (uint64_t)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Mahalanobis form in the reference's op order (forward.py:101-105):
//   q = a00*dx^2 + (2*a01)*dx*dy + a11*dy^2, left to right, no FMA.
__device__ __forceinline__ double quadform(double a00, double a01, double a11,
                                           double dx, double dy) {
  double t1 = dmul(a00, dmul(dx, dx));
  double t2 = dmul(dmul(dmul(2.0, a01), dx), dy);
  double t3 = dmul(a11, dmul(dy, dy));
  return dadd(dadd(t1, t2), t3);
}

// 256-bit in-tile member mask of one Gaussian (bit = local cell (iv&15)*16+(iu&15)).
// Small footprints: the 8x8 window rows are shifted into place (no per-bit
// loop).  Large footprints: exact FP64 test of the bbox cells in the tile.
__device__ __forceinline__ void member_mask(double u, double v, double a00, double a01, double a11,
                                            uint64_t cell_mask, int x0, int x1, int y0, int y1, int tx, int ty,
                                            double cutoff, uint64_t m[4]) {
  m[0] = m[1] = m[2] = m[3] = 0;
  if (x0 > x1 || y0 > y1) return;
  if ((x1 - x0) < 8 && (y1 - y0) < 8) {
    const uint64_t cm = cell_mask;
    const int c0 = x0 - tx * kTile, r0 = y0 - ty * kTile;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int rr = r0 + k;
      const uint32_t byte = (uint32_t)(cm >> (8 * k)) & 0xffu;
      if (rr < 0 || rr > 15 || byte == 0) continue;
      const uint32_t bits = (c0 >= 0 ? (byte << c0) : (byte >> (-c0))) & 0xffffu;
      const uint64_t v = (uint64_t)bits << ((rr & 3) * 16);
      const int w = rr >> 2;
#pragma unroll
      for (int q = 0; q < 4; ++q) m[q] |= (w == q) ? v : 0ull;
    }
    return;
  }
  const bool dense = !isfinite(cutoff);
  const double cut2 = dmul(cutoff, cutoff), a01x2 = dmul(2.0, a01);
  const int cx0 = max(x0, tx * kTile), cx1 = min(x1, tx * kTile + kTile - 1);
  const int cy0 = max(y0, ty * kTile), cy1 = min(y1, ty * kTile + kTile - 1);
  for (int iv = cy0; iv <= cy1; ++iv) {
    const double dy = dsub((double)iv, v);
    const double t3 = dmul(a11, dmul(dy, dy));
    for (int iu = cx0; iu <= cx1; ++iu) {
      bool member = dense;
      if (!dense) {
        const double dx = dsub((double)iu, u);
        const double q = dadd(dadd(dmul(a00, dmul(dx, dx)), dmul(dmul(a01x2, dx), dy)), t3);
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

__device__ __forceinline__ void member_mask(const sdgr_pair_rec& r, int tx, int ty, double cutoff, uint64_t m[4]) {
  member_mask(r.u, r.v, r.a00, r.a01, r.a11, r.cell_mask, r.x0, r.x1, r.y0, r.y1, tx, ty, cutoff, m);
}

__device__ __forceinline__ double softplus64(double x) {
  // np.logaddexp(0, x) = max(x,0) + log1p(exp(-|x|))  (scene.py:22-25)
  if (!(x == x)) return x;
  return fmax(x, 0.0) + log1p(exp(-fabs(x)));
}

// Launch accounting (sdgr_launch_count).
void note_launch(int n = 1);
int check_launch();  // returns SDGR_OK or SDGR_ERR_CUDA after a launch

// Kernel timing (sdgr_profile_begin/end): events around a launch, only when
// the kernel's bit is enabled.  Usage: { KernelTimer kt(SDGR_K_WALK, st); k<<<...>>>(...); }
void prof_mark(int id, bool begin, cudaStream_t st);
struct KernelTimer {
  int id;
  cudaStream_t st;
  KernelTimer(int i, cudaStream_t s) : id(i), st(s) { prof_mark(id, true, st); }
  ~KernelTimer() { prof_mark(id, false, st); }
};

template <typename T>
__device__ __forceinline__ T ldg(const T* p) { return __ldg(p); }

// SMs of the current device (cached; persistent grids are sized from it)
inline int sm_count() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

}  // namespace sdgr
