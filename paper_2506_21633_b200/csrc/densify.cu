// densify.cu — densification bookkeeping on the device:
//   k_accum_update    GradAccumulator.update (optimize.py:229-233)
//   k_densify_flags   the clone / split decisions of densify_and_prune
//                     (optimize.py:266-271)
//   k_clone_shift     clones move one position-lr step down the mean
//                     position gradient (optimize.py:276-279)
//   k_split_children  children sample inside the parent footprint:
//                     x += chol(Sigma) xi, log-scales shrink
//                     (optimize.py:282-289; xi from the caller's RNG)
//   k_prune_flags     survivors: DC phase above the floor, not oversized
//                     (optimize.py:293-296)
// Row compaction (select / concatenate) is a gather the caller performs with
// the index lists these flags define; the random draws stay on the host so
// the same seeded generator gives the reference's children bit for bit.
#include "common.cuh"

namespace sdgr {

template <typename T>
__device__ __forceinline__ double ld(const void* p, int64_t i) {
  return (double)static_cast<const T*>(p)[i];
}

__global__ void __launch_bounds__(256) k_accum_update(sdgr_grads gr, int64_t n, double* __restrict__ norm_sum,
                                                      double* __restrict__ pos_sum, double* __restrict__ count) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  // views in which g was visible (1 per single-view backward)
  const int vis = gr.visible_dtype ? (int)static_cast<const float*>(gr.visible)[g]
                                   : static_cast<const int32_t*>(gr.visible)[g];
  if (vis <= 0) return;
  norm_sum[g] += (double)static_cast<const float*>(gr.uv_grad_norm)[g];
  for (int k = 0; k < 3; ++k) pos_sum[3 * g + k] += (double)static_cast<const float*>(gr.positions)[3 * g + k];
  count[g] += (double)vis;
}

// max over the three axes of exp(log_scale)
template <typename T>
__device__ __forceinline__ double max_scale(const sdgr_scene& s, int64_t g) {
  const double a = exp(ld<T>(s.log_scales, 3 * g)), b = exp(ld<T>(s.log_scales, 3 * g + 1)),
               c = exp(ld<T>(s.log_scales, 3 * g + 2));
  return fmax(fmax(a, b), c);
}

template <typename T>
__global__ void __launch_bounds__(256) k_densify_flags(sdgr_scene s, const double* __restrict__ norm_sum,
                                                       const double* __restrict__ count, double cap,
                                                       double small_size, double grad_thr,
                                                       uint8_t* __restrict__ flags) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= s.n) return;
  const double ms = max_scale<T>(s, g);
  const bool split = ms > cap;
  const bool small = ms <= small_size;
  const double mean_norm = norm_sum[g] / fmax(count[g], 1.0);
  const bool clone = mean_norm > grad_thr && small && !split && count[g] > 0.0;
  flags[g] = split ? 2 : (clone ? 1 : 0);
}

// rows already gathered (clones in selection order): positions += -lr * pos_sum / max(count, 1)
template <typename T>
__global__ void __launch_bounds__(256) k_clone_shift(sdgr_scene c, const double* __restrict__ pos_sum,
                                                     const double* __restrict__ count, double lr) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= c.n) return;
  T* P = (T*)c.positions;
  const double den = fmax(count[g], 1.0);
  for (int k = 0; k < 3; ++k) {
    const double disp = -lr * (pos_sum[3 * g + k] / den);
    P[3 * g + k] = (T)((double)P[3 * g + k] + disp);
  }
}

// children (parent rows, each twice): x += L xi with L L^T = Sigma = M M^T,
// M = R(q_hat) diag(e^s); log-scales -= log(shrink)
template <typename T>
__global__ void __launch_bounds__(256) k_split_children(sdgr_scene c, const double* __restrict__ xi,
                                                        double log_shrink) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= c.n) return;
  double q[4];
  for (int k = 0; k < 4; ++k) q[k] = ld<T>(c.rotations, 4 * g + k);
  const double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double w = q[0] / nrm, x = q[1] / nrm, y = q[2] / nrm, z = q[3] / nrm;
  const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                       2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                       2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
  double sc[3], M[9], S[9];
  for (int j = 0; j < 3; ++j) sc[j] = exp(ld<T>(c.log_scales, 3 * g + j));
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M[3 * i + j] = R[3 * i + j] * sc[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) S[3 * i + j] = M[3 * i] * M[3 * j] + M[3 * i + 1] * M[3 * j + 1] + M[3 * i + 2] * M[3 * j + 2];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < i; ++j) S[3 * i + j] = S[3 * j + i] = 0.5 * (S[3 * i + j] + S[3 * j + i]);
  // lower Cholesky factor
  const double l00 = sqrt(S[0]);
  const double l10 = S[3] / l00, l20 = S[6] / l00;
  const double l11 = sqrt(S[4] - l10 * l10);
  const double l21 = (S[7] - l20 * l10) / l11;
  const double l22 = sqrt(S[8] - l20 * l20 - l21 * l21);
  const double x0 = xi[3 * g], x1 = xi[3 * g + 1], x2 = xi[3 * g + 2];
  const double d[3] = {l00 * x0, l10 * x0 + l11 * x1, l20 * x0 + l21 * x1 + l22 * x2};
  T* P = (T*)c.positions;
  T* L = (T*)c.log_scales;
  for (int k = 0; k < 3; ++k) {
    P[3 * g + k] = (T)((double)P[3 * g + k] + d[k]);
    L[3 * g + k] = (T)((double)L[3 * g + k] - log_shrink);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_prune_flags(sdgr_scene s, double cap, double phase_floor, double sh_c0,
                                                     uint8_t* __restrict__ survive) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= s.n) return;
  const double dc = ld<T>(s.sh_coeffs, 16 * g) * sh_c0;
  survive[g] = (dc >= phase_floor && !(max_scale<T>(s, g) > cap)) ? 1 : 0;
}

#define SDGR_DISPATCH(sc, KERNEL, ...)                                             \
  do {                                                                             \
    const unsigned blocks_ = (unsigned)(((sc).n + 255) / 256);                     \
    if ((sc).dtype == 0) KERNEL<float><<<blocks_, 256, 0, st>>>(__VA_ARGS__);      \
    else KERNEL<double><<<blocks_, 256, 0, st>>>(__VA_ARGS__);                     \
  } while (0)

int launch_accum_update(const sdgr_grads& gr, int64_t n, double* norm_sum, double* pos_sum, double* count,
                        cudaStream_t st) {
  k_accum_update<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(gr, n, norm_sum, pos_sum, count);
  note_launch();
  return check_launch();
}

int launch_densify_flags(const sdgr_scene& s, const double* norm_sum, const double* count, double cap,
                         double small_size, double grad_thr, uint8_t* flags, cudaStream_t st) {
  SDGR_DISPATCH(s, k_densify_flags, s, norm_sum, count, cap, small_size, grad_thr, flags);
  note_launch();
  return check_launch();
}

int launch_clone_shift(const sdgr_scene& c, const double* pos_sum, const double* count, double lr,
                       cudaStream_t st) {
  SDGR_DISPATCH(c, k_clone_shift, c, pos_sum, count, lr);
  note_launch();
  return check_launch();
}

int launch_split_children(const sdgr_scene& c, const double* xi, double log_shrink, cudaStream_t st) {
  SDGR_DISPATCH(c, k_split_children, c, xi, log_shrink);
  note_launch();
  return check_launch();
}

int launch_prune_flags(const sdgr_scene& s, double cap, double phase_floor, double sh_c0, uint8_t* survive,
                       cudaStream_t st) {
  SDGR_DISPATCH(s, k_prune_flags, s, cap, phase_floor, sh_c0, survive);
  note_launch();
  return check_launch();
}

}  // namespace sdgr
