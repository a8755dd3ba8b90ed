// plyio.cu — scene checkpoints in the reference's binary PLY layout
// (ply.py:36-49, save_scene :110-123, load_scene :126-155; SURVEY.md §8f row
// 3): one vertex per Gaussian, 28 little-endian doubles in SCENE_PROPERTIES
// order.  The vertex-major interleave (pack) and its inverse (unpack, with a
// column map so files with reordered or extra double properties load) run on
// the device, so a 1M-Gaussian checkpoint moves as one 224 MB copy.
#include "common.cuh"

namespace sdgr {

constexpr int kPlyCols = 28;
struct PlyMap {
  int32_t col[kPlyCols];  // column of scene property k within a vertex record
};

// scene property k -> (group pointer, width, component)
template <typename T>
__device__ __forceinline__ T* prop_ptr(const sdgr_scene& s, int k, int64_t g) {
  if (k < 3) return (T*)s.positions + 3 * g + k;
  if (k < 7) return (T*)s.rotations + 4 * g + (k - 3);
  if (k < 10) return (T*)s.log_scales + 3 * g + (k - 7);
  if (k < 26) return (T*)s.sh_coeffs + 16 * g + (k - 10);
  return (T*)s.ke_raw + 2 * g + (k - 26);
}

template <typename T>
__global__ void __launch_bounds__(256) k_ply_pack(sdgr_scene s, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one output double
  if (i >= s.n * kPlyCols) return;
  const int64_t g = i / kPlyCols;
  const int k = (int)(i % kPlyCols);
  out[i] = (double)*prop_ptr<T>(s, k, g);
}

template <typename T>
__global__ void __launch_bounds__(256) k_ply_unpack(const double* __restrict__ in, int64_t n, int stride,
                                                    PlyMap map, sdgr_scene s) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * kPlyCols) return;
  const int64_t g = i / kPlyCols;
  const int k = (int)(i % kPlyCols);
  *prop_ptr<T>(s, k, g) = (T)in[g * stride + map.col[k]];
}

int launch_ply_pack(const sdgr_scene& s, double* out, cudaStream_t st) {
  const unsigned blocks = (unsigned)((s.n * kPlyCols + 255) / 256);
  if (s.dtype == 0) k_ply_pack<float><<<blocks, 256, 0, st>>>(s, out);
  else k_ply_pack<double><<<blocks, 256, 0, st>>>(s, out);
  note_launch();
  return check_launch();
}

int launch_ply_unpack(const double* in, int64_t n, int stride, const int32_t* col, const sdgr_scene& s,
                      cudaStream_t st) {
  PlyMap m;
  for (int k = 0; k < kPlyCols; ++k) m.col[k] = col[k];
  const unsigned blocks = (unsigned)((n * kPlyCols + 255) / 256);
  if (s.dtype == 0) k_ply_unpack<float><<<blocks, 256, 0, st>>>(in, n, stride, m, s);
  else k_ply_unpack<double><<<blocks, 256, 0, st>>>(in, n, stride, m, s);
  note_launch();
  return check_launch();
}

}  // namespace sdgr
