// train.cu — the steps either side of the path in the reference's training
// loop, on the device so a whole optimiser step needs no
// host round trip:
//   loss   optimize.loss (optimize.py:85-102): (1-l) mean|S-Y| + l (1-SSIM)
//          and dL/dS, SSIM with its analytic gradient (metrics.py:98-137):
//          11x11 Gaussian window (sigma 1.5), separable, zero padded, value
//          averaged over the interior where the window fits; images smaller
//          than the window use one global window (metrics.py:60-62, 117-121).
//   adam   optimize.adam_step (optimize.py:171-207): non-finite gradient
//          entries zeroed and counted, bias-corrected moments, position steps
//          norm-clamped to the displacement bound, quaternions renormalised.
// FP64 throughout; reductions are fixed-order (per-block partials summed in
// block order by one block), so values are run-to-run deterministic.
#include "common.cuh"

namespace sdgr {

constexpr int kWin = 11, kRad = 5;
constexpr int kRedBlocks = 256;  // partial sums per reduction

struct SsimKernel {
  double w[kWin];
};

// vertical (axis 0) correlation of n_in images; in images are computed from
// x, y by `which` (0 x, 1 y, 2 x*x, 3 y*y, 4 x*y) when src == nullptr
__global__ void __launch_bounds__(256) k_filter_v(const double* __restrict__ x, const double* __restrict__ y,
                                                  const double* __restrict__ src, int n_img, int h, int w,
                                                  SsimKernel K, double* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t hw = (int64_t)h * w;
  if (p >= hw) return;
  const int i = (int)(p / w), j = (int)(p % w);
  for (int m = 0; m < n_img; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < kWin; ++t) {
      const int ii = i + t - kRad;
      if (ii < 0 || ii >= h) continue;
      const int64_t q = (int64_t)ii * w + j;
      double v;
      if (src) {
        v = src[m * hw + q];
      } else {
        const double a = x[q], b = y[q];
        v = m == 0 ? a : m == 1 ? b : m == 2 ? a * a : m == 3 ? b * b : a * b;
      }
      acc += K.w[t] * v;
    }
    out[m * hw + p] = acc;
  }
}

// horizontal (axis 1) correlation
__global__ void __launch_bounds__(256) k_filter_h(const double* __restrict__ in, int n_img, int h, int w,
                                                  SsimKernel K, double* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t hw = (int64_t)h * w;
  if (p >= hw) return;
  const int i = (int)(p / w), j = (int)(p % w);
  for (int m = 0; m < n_img; ++m) {
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < kWin; ++t) {
      const int jj = j + t - kRad;
      if (jj < 0 || jj >= w) continue;
      acc += K.w[t] * in[m * hw + (int64_t)i * w + jj];
    }
    out[m * hw + p] = acc;
  }
}

// deterministic block partial sums of up to 4 per-element quantities
template <int NQ>
__device__ __forceinline__ void block_partials(const double (&v)[NQ], double* partials) {
  __shared__ double sh[NQ][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double s[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    s[q] = v[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s[q] += __shfl_down_sync(0xffffffffu, s[q], off);
    if (lane == 0) sh[q][warp] = s[q];
  }
  __syncthreads();
  if (threadIdx.x < NQ) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[threadIdx.x][k];
    partials[threadIdx.x * kRedBlocks + blockIdx.x] = t;
  }
}

// SSIM map pieces -> weighted partial-derivative images + partial sums of
// the interior SSIM and of |x - y|.  mom: ux, uy, ex2, ey2, exy.
__global__ void __launch_bounds__(256) k_ssim_map(const double* __restrict__ x, const double* __restrict__ y,
                                                  const double* __restrict__ mom, int h, int w, double c1,
                                                  double c2, double inv_nwin, double* __restrict__ dimg,
                                                  double* __restrict__ partials) {
  const int64_t hw = (int64_t)h * w;
  double sm = 0.0, l1 = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < hw; p += (int64_t)gridDim.x * blockDim.x) {
    const double ux = mom[p], uy = mom[hw + p], ex2 = mom[2 * hw + p], ey2 = mom[3 * hw + p],
                 exy = mom[4 * hw + p];
    const double vx = ex2 - ux * ux, vy = ey2 - uy * uy, cxy = exy - ux * uy;
    const double a1 = 2.0 * ux * uy + c1, a2 = 2.0 * cxy + c2;
    const double b1 = ux * ux + uy * uy + c1, b2 = vx + vy + c2;
    const double denom = b1 * b2;
    const double smap = (a1 * a2) / denom;
    const int i = (int)(p / w), j = (int)(p % w);
    const bool interior = i >= kRad && i < h - kRad && j >= kRad && j < w - kRad;
    const double wt = interior ? inv_nwin : 0.0;
    if (interior) sm += smap;
    l1 += fabs(x[p] - y[p]);
    const double ds_da1 = a2 / denom, ds_da2 = a1 / denom;
    const double ds_db1 = -smap / b1, ds_db2 = -smap / b2;
    const double ds_dux = ds_da1 * 2.0 * uy + ds_da2 * (-2.0 * uy) + ds_db1 * 2.0 * ux + ds_db2 * (-2.0 * ux);
    dimg[p] = wt * ds_dux;
    dimg[hw + p] = wt * ds_db2;
    dimg[2 * hw + p] = wt * (ds_da2 * 2.0);
  }
  const double v[2] = {sm, l1};
  block_partials<2>(v, partials);
}

// grad = (1-l) sign(x-y)/n - l (B0 + 2 x B1 + y B2), B = back-filtered images
__global__ void __launch_bounds__(256) k_loss_grad(const double* __restrict__ x, const double* __restrict__ y,
                                                   const double* __restrict__ back, int64_t hw, double lam,
                                                   double* __restrict__ grad) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= hw) return;
  const double d = x[p] - y[p];
  const double sgn = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
  double g = sgn / (double)hw * (1.0 - lam);
  if (back) g -= lam * (back[p] + 2.0 * x[p] * back[hw + p] + y[p] * back[2 * hw + p]);
  grad[p] = g;
}

// value = (1-l) L1 + l (1 - SSIM) from the partial sums (one block, in order)
__global__ void k_loss_value(const double* __restrict__ partials, int64_t hw, double inv_nwin, double lam,
                             int ssim_q, double* __restrict__ value) {
  if (threadIdx.x != 0) return;
  double sm = 0.0, l1 = 0.0;
  for (int b = 0; b < kRedBlocks; ++b) {
    if (ssim_q >= 0) sm += partials[ssim_q * kRedBlocks + b];
    l1 += partials[kRedBlocks + b];
  }
  double v = (1.0 - lam) * (l1 / (double)hw);
  if (ssim_q >= 0) v += lam * (1.0 - sm * inv_nwin);
  *value = v;
}

// ---- global-window SSIM (images smaller than the window, metrics.py:60-62)
__global__ void __launch_bounds__(256) k_global_moments(const double* __restrict__ x, const double* __restrict__ y,
                                                        int64_t hw, double* __restrict__ partials) {
  double s[4] = {0, 0, 0, 0};
  double sxy = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < hw; p += (int64_t)gridDim.x * blockDim.x) {
    const double a = x[p], b = y[p];
    s[0] += a; s[1] += b; s[2] += a * a; s[3] += b * b;
    sxy += a * b;
  }
  block_partials<4>(s, partials);
  __syncthreads();
  const double v[2] = {sxy, 0.0};
  block_partials<2>(v, partials + 4 * kRedBlocks);
}

// one block: the global-window SSIM value and its three gradient scalars
__global__ void k_global_ssim(const double* __restrict__ partials, int64_t hw, double c1, double c2,
                              double* __restrict__ gs) {
  if (threadIdx.x != 0) return;
  double m[5] = {0, 0, 0, 0, 0};
  for (int q = 0; q < 5; ++q)
    for (int b = 0; b < kRedBlocks; ++b) m[q] += partials[q * kRedBlocks + b];
  const double n = (double)hw;
  const double ux = m[0] / n, uy = m[1] / n, ex2 = m[2] / n, ey2 = m[3] / n, exy = m[4] / n;
  const double vx = ex2 - ux * ux, vy = ey2 - uy * uy, cxy = exy - ux * uy;
  const double a1 = 2.0 * ux * uy + c1, a2 = 2.0 * cxy + c2;
  const double b1 = ux * ux + uy * uy + c1, b2 = vx + vy + c2;
  const double denom = b1 * b2;
  const double smap = (a1 * a2) / denom;
  const double ds_da1 = a2 / denom, ds_da2 = a1 / denom;
  const double ds_db1 = -smap / b1, ds_db2 = -smap / b2;
  const double wt = 1.0 / n;
  const double ds_dux = ds_da1 * 2.0 * uy + ds_da2 * (-2.0 * uy) + ds_db1 * 2.0 * ux + ds_db2 * (-2.0 * ux);
  // back(z) = full(sum(z) / n) with z = wt * const -> each is wt * const
  gs[0] = smap;
  gs[1] = (wt * ds_dux) * n / n;
  gs[2] = (wt * ds_db2) * n / n;
  gs[3] = (wt * (ds_da2 * 2.0)) * n / n;
}

__global__ void __launch_bounds__(256) k_loss_grad_global(const double* __restrict__ x,
                                                          const double* __restrict__ y, const double* gs,
                                                          const double* __restrict__ partials, int64_t hw,
                                                          double lam, double* __restrict__ grad,
                                                          double* __restrict__ value) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0) {
    double l1 = 0.0;
    for (int b = 0; b < kRedBlocks; ++b) l1 += partials[5 * kRedBlocks + b];
    *value = (1.0 - lam) * (l1 / (double)hw) + lam * (1.0 - gs[0]);
  }
  if (p >= hw) return;
  const double d = x[p] - y[p];
  const double sgn = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
  grad[p] = sgn / (double)hw * (1.0 - lam) - lam * (gs[1] + 2.0 * x[p] * gs[2] + y[p] * gs[3]);
}

__global__ void __launch_bounds__(256) k_abs_partials(const double* __restrict__ x, const double* __restrict__ y,
                                                      int64_t hw, double* __restrict__ partials) {
  double l1 = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < hw; p += (int64_t)gridDim.x * blockDim.x)
    l1 += fabs(x[p] - y[p]);
  const double v[1] = {l1};
  block_partials<1>(v, partials);
}

size_t loss_scratch_bytes(int h, int w) {
  const size_t hw = (size_t)h * w;
  return sizeof(double) * (5 * hw + 5 * hw + 3 * hw + 3 * hw + 6 * kRedBlocks + 8);
}

int launch_loss(const double* S, const double* Y, int h, int w, double lam, double max_val,
                const double* kernel11, double* value, double* grad, void* scratch, cudaStream_t st) {
  const int64_t hw = (int64_t)h * w;
  const unsigned blocks = (unsigned)((hw + 255) / 256);
  double* tmp = static_cast<double*>(scratch);  // 5 hw
  double* mom = tmp + 5 * hw;                    // 5 hw
  double* dimg = mom + 5 * hw;                   // 3 hw
  double* back = dimg + 3 * hw;                  // 3 hw
  double* partials = back + 3 * hw;              // 6 * kRedBlocks
  double* gs = partials + 6 * kRedBlocks;        // 4
  const double c1 = (0.01 * max_val) * (0.01 * max_val), c2 = (0.03 * max_val) * (0.03 * max_val);
  if (lam <= 0.0) {
    k_abs_partials<<<kRedBlocks, 256, 0, st>>>(S, Y, hw, partials + kRedBlocks);
    k_loss_value<<<1, 32, 0, st>>>(partials, hw, 0.0, lam, -1, value);
    k_loss_grad<<<blocks, 256, 0, st>>>(S, Y, nullptr, hw, lam, grad);
    note_launch(3);
    return check_launch();
  }
  if (h >= kWin && w >= kWin) {
    SsimKernel K;
    for (int t = 0; t < kWin; ++t) K.w[t] = kernel11[t];
    const double inv_nwin = 1.0 / ((double)(h - 2 * kRad) * (double)(w - 2 * kRad));
    k_filter_v<<<blocks, 256, 0, st>>>(S, Y, nullptr, 5, h, w, K, tmp);
    k_filter_h<<<blocks, 256, 0, st>>>(tmp, 5, h, w, K, mom);
    k_ssim_map<<<kRedBlocks, 256, 0, st>>>(S, Y, mom, h, w, c1, c2, inv_nwin, dimg, partials);
    k_filter_v<<<blocks, 256, 0, st>>>(nullptr, nullptr, dimg, 3, h, w, K, tmp);
    k_filter_h<<<blocks, 256, 0, st>>>(tmp, 3, h, w, K, back);
    k_loss_grad<<<blocks, 256, 0, st>>>(S, Y, back, hw, lam, grad);
    k_loss_value<<<1, 32, 0, st>>>(partials, hw, inv_nwin, lam, 0, value);
    note_launch(7);
  } else {
    k_global_moments<<<kRedBlocks, 256, 0, st>>>(S, Y, hw, partials);
    k_abs_partials<<<kRedBlocks, 256, 0, st>>>(S, Y, hw, partials + 5 * kRedBlocks);
    k_global_ssim<<<1, 32, 0, st>>>(partials, hw, c1, c2, gs);
    k_loss_grad_global<<<blocks, 256, 0, st>>>(S, Y, gs, partials, hw, lam, grad, value);
    note_launch(4);
  }
  return check_launch();
}

// ======================================================================= Adam
struct AdamArgs {
  double lr[5];
  double b1, b2, eps, bc1, bc2;
  double bound;  // <= 0: no displacement clamp
};

template <typename T>
__device__ __forceinline__ double adam_one(T* param, T* m, T* v, const void* grad_, int64_t i, const AdamArgs& A,
                                           double lr, unsigned long long& bad) {
  double g = (double)static_cast<const float*>(grad_)[i];
  if (!isfinite(g)) {
    ++bad;
    g = 0.0;
  }
  // numpy's order, no contraction: m = m*b1 + (1-b1)*g; v = v*b2 + ((1-b2)*g)*g
  const double mm = dadd(dmul((double)m[i], A.b1), dmul(dsub(1.0, A.b1), g));
  const double vv = dadd(dmul((double)v[i], A.b2), dmul(dmul(dsub(1.0, A.b2), g), g));
  m[i] = (T)mm;
  v[i] = (T)vv;
  // step = lr * (m / bc1) / (sqrt(v / bc2) + eps)
  return ddiv(dmul(lr, ddiv(mm, A.bc1)), dadd(dsqrt(ddiv(vv, A.bc2)), A.eps));
}

template <typename T>
__global__ void __launch_bounds__(256) k_adam(sdgr_scene sc, sdgr_grads gr, sdgr_scene m, sdgr_scene v,
                                              AdamArgs A, unsigned long long* n_skipped,
                                              const int32_t* guard) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long bad = 0;
  if (guard && *guard) return;  // overflowed step: its gradients are truncated
  if (g < sc.n) {
    // positions: per-row displacement clamp (optimize.py:196-199)
    {
      T* P = (T*)(sc.positions);
      double st[3];
      for (int k = 0; k < 3; ++k)
        st[k] = adam_one<T>(P, (T*)(m.positions), (T*)(v.positions), gr.positions,
                            3 * g + k, A, A.lr[0], bad);
      if (A.bound > 0.0) {
        const double nrm = dsqrt(dadd(dadd(dmul(st[0], st[0]), dmul(st[1], st[1])), dmul(st[2], st[2])));
        const double f = fmin(1.0, ddiv(A.bound, fmax(nrm, 1e-300)));
        for (int k = 0; k < 3; ++k) st[k] = dmul(st[k], f);
      }
      for (int k = 0; k < 3; ++k) P[3 * g + k] = (T)dsub((double)P[3 * g + k], st[k]);
    }
    // rotations, then the renormalisation (optimize.py:207)
    {
      T* R = (T*)(sc.rotations);
      double q[4];
      for (int k = 0; k < 4; ++k) {
        const double s = adam_one<T>(R, (T*)(m.rotations), (T*)(v.rotations), gr.rotations,
                                     4 * g + k, A, A.lr[1], bad);
        q[k] = (double)(T)dsub((double)R[4 * g + k], s);
      }
      const double nrm =
          dsqrt(dadd(dadd(dadd(dmul(q[0], q[0]), dmul(q[1], q[1])), dmul(q[2], q[2])), dmul(q[3], q[3])));
      for (int k = 0; k < 4; ++k) R[4 * g + k] = (T)ddiv(q[k], nrm);
    }
    auto group = [&](const void* p, const void* mp, const void* vp, const void* gp, int width, double lr) {
      T* P = (T*)(p);
      for (int k = 0; k < width; ++k) {
        const int64_t i = (int64_t)width * g + k;
        const double s = adam_one<T>(P, (T*)(mp), (T*)(vp), gp, i, A, lr, bad);
        P[i] = (T)dsub((double)P[i], s);
      }
    };
    group(sc.log_scales, m.log_scales, v.log_scales, gr.log_scales, 3, A.lr[2]);
    group(sc.sh_coeffs, m.sh_coeffs, v.sh_coeffs, gr.sh_coeffs, 16, A.lr[3]);
    group(sc.ke_raw, m.ke_raw, v.ke_raw, gr.ke_raw, 2, A.lr[4]);
  }
  // integer counts: associative, so the total is deterministic
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) bad += __shfl_down_sync(0xffffffffu, bad, off);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(n_skipped, bad);
}

int launch_adam(const sdgr_scene& sc, const sdgr_grads& gr, const sdgr_scene& m, const sdgr_scene& v,
                const double* lr, double b1, double b2, double eps, double bc1, double bc2, double bound,
                unsigned long long* n_skipped, const int32_t* guard, cudaStream_t st) {
  AdamArgs A;
  for (int k = 0; k < 5; ++k) A.lr[k] = lr[k];
  A.b1 = b1; A.b2 = b2; A.eps = eps; A.bc1 = bc1; A.bc2 = bc2; A.bound = bound;
  const unsigned blocks = (unsigned)((sc.n + 255) / 256);
  if (sc.dtype == 0)
    k_adam<float><<<blocks, 256, 0, st>>>(sc, gr, m, v, A, n_skipped, guard);
  else
    k_adam<double><<<blocks, 256, 0, st>>>(sc, gr, m, v, A, n_skipped, guard);
  note_launch();
  return check_launch();
}

}  // namespace sdgr
